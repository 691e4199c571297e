// Instantiates the 1/4/3 networks (RN/RZ x gradual/FTZ); see bfp_formats.h.
#include "../bfp_kernels.cuh"
BFP_INSTANTIATE(4, 3)

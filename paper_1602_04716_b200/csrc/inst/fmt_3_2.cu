// Instantiates the 1/3/2 networks (RN/RZ x gradual/FTZ); see bfp_formats.h.
#include "../bfp_kernels.cuh"
BFP_INSTANTIATE(3, 2)

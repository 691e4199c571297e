// Instantiates the 1/5/7 networks (RN/RZ x gradual/FTZ); see bfp_formats.h.
#include "../bfp_kernels.cuh"
BFP_INSTANTIATE(5, 7)

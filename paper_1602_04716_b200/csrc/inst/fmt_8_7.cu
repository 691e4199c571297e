// Instantiates the 1/8/7 networks (RN/RZ x gradual/FTZ); see bfp_formats.h.
#include "../bfp_kernels.cuh"
BFP_INSTANTIATE(8, 7)

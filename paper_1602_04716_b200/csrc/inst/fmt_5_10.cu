// Instantiates the 1/5/10 networks (RN/RZ x gradual/FTZ); see bfp_formats.h.
#include "../bfp_kernels.cuh"
BFP_INSTANTIATE(5, 10)

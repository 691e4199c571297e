// bfp_probe.cu -- LOP3 issue-rate probe: the logic leg of the roofline is
// measured on the box, not assumed.  8 independent LOP3
// chains per thread, volatile so ptxas keeps every instruction; the grid
// fills every SM.
#include <cuda_runtime.h>

#include <cstdint>

#include "../../include/bfpgpu.h"

namespace {

__global__ void __launch_bounds__(256) k_lop3_peak(uint32_t* out, int iters) {
  uint32_t a[8];
  const uint32_t b = threadIdx.x * 0x9e3779b9u, c = blockIdx.x * 0x85ebca6bu;
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = threadIdx.x + j * 0x01000193u;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
#pragma unroll
      for (int j = 0; j < 8; ++j)
        asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(a[j]) : "r"(a[(j + 1) & 7]), "r"(k & 1 ? b : c));
    }
  }
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) r ^= a[j];
  if (r == 0x12345678u) out[0] = r;
}

}  // namespace

extern "C" bfp_status bfp_probe_lop3(int iters, float* ms, double* lop3_per_s) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  uint32_t* out = nullptr;
  if (cudaMalloc(&out, 4) != cudaSuccess) return BFP_ECUDA;
  const int grid = sms * 8, threads = 256;
  k_lop3_peak<<<grid, threads>>>(out, 4);  // warm-up
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_lop3_peak<<<grid, threads>>>(out, iters);
  cudaEventRecord(e1);
  cudaError_t err = cudaEventSynchronize(e1);
  float t = 0;
  cudaEventElapsedTime(&t, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  if (err != cudaSuccess) return BFP_ECUDA;
  if (ms) *ms = t;
  if (lop3_per_s) *lop3_per_s = double(grid) * threads * iters * 16.0 * 8.0 / (t * 1e-3);
  return BFP_OK;
}

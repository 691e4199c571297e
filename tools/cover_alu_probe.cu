// tools/cover_alu_probe.cu -- how busy can the ALU pipe get on a cover ALONE?
// Runs a generated LOP3 cover (default: the 1/6/9 fused mul_add of config 5) in
// registers with its operands re-read from a 16 KiB cache-resident buffer, at the shipped kernel's
// occupancy (128-thread CTAs, __launch_bounds__(128, MINB)).  Under
//   ncu --metrics sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
// the pipe utilisation it reaches is the ceiling the instruction stream itself
// allows (dependencies, register banks, issue); what the streaming kernel
// loses against it is the memory side.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr \
//        -Ipaper_1602_04716_b200/csrc tools/cover_alu_probe.cu -o tools/cover_alu_probe
//   tools/cover_alu_probe [iters]
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>

#include "bfp_circuits.cuh"
#include "gen/gen_6_9.cuh"
#include "gen/gen_8_15.cuh"

using namespace bfpg;

template <class F, int OP, int MINB>
__global__ void __launch_bounds__(128, MINB) k_cover_only(w32* out, const w32* seed, int iters) {
  constexpr int N = F::N;
  const unsigned t = blockIdx.x * blockDim.x + threadIdx.x;
  w32 r = 0;
  for (int i = 0; i < iters; ++i) {
    // the unit's operands come from a 16 KiB buffer (L1 hits after the first
    // touch): the register profile of the streaming kernel -- operands die as
    // the network consumes them -- without its DRAM latency
    w32 X[N], Y[N], C[N], Z[N];
    const unsigned b = (t + unsigned(i) * 97u) & 1023u;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      X[j] = __ldg(seed + ((b + j * 32) & 4095));
      Y[j] = __ldg(seed + ((b + j * 32 + 1024) & 4095));
      C[j] = __ldg(seed + ((b + j * 32 + 2048) & 4095));
    }
    Gen<F, OP>::run(X, Y, C, Z);
#pragma unroll
    for (int j = 0; j < N; ++j) r ^= Z[j];  // N extra LOP3-class ops per unit
  }
  out[t] = r;
}

template <class F, int OP, int MINB>
void run(const char* name, int iters) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * MINB, threads = 128;
  w32 *out, *seed;
  cudaMalloc(&out, size_t(grid) * threads * 4);
  cudaMalloc(&seed, 4096 * 4);
  w32 h[4096];
  unsigned long long s = 0x9E3779B97F4A7C15ull;
  for (int i = 0; i < 4096; ++i) {
    s = s * 6364136223846793005ull + 1442695040888963407ull;
    h[i] = w32(s >> 32);
  }
  cudaMemcpy(seed, h, sizeof h, cudaMemcpyHostToDevice);
  k_cover_only<F, OP, MINB><<<grid, threads>>>(out, seed, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  k_cover_only<F, OP, MINB><<<grid, threads>>>(out, seed, iters);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double luts = Gen<F, OP>::luts + F::N;
  const double rate = double(grid) * threads * iters * luts / (ms * 1e-3);
  std::printf("%s: %d CTAs/SM, %d LUTs + %d feedback per unit, %d iters: %.3f ms, %.2f T LOP3/s, %.1f Gelem/s equivalent\n",
              name, MINB, Gen<F, OP>::luts, F::N, iters, ms, rate * 1e-12,
              double(grid) * threads * iters * 32.0 / (ms * 1e-3) * 1e-9);
  cudaFree(out);
  cudaFree(seed);
}

int main(int argc, char** argv) {
  const int iters = argc > 1 ? std::atoi(argv[1]) : 2000;
  run<Format<6, 9, true, false>, 4, 5>("1/6/9 mul_add", iters);
  run<Format<6, 9, true, false>, 4, 4>("1/6/9 mul_add", iters);
  run<Format<8, 15, true, false>, 2, 4>("1/8/15 mul", iters);
  return 0;
}

// bfp_kernels.cuh -- sm_100a kernels over the slice-major plane layout.
//
// Arithmetic (add / sub / mul / div / mul_add): one thread per 32-element unit.
// A warp owns one 1024-element block: for every plane the 32 threads read 32
// consecutive words (one 128-B line), evaluate the format's unrolled LOP3
// network in registers and write 32 consecutive words.  Loads use the
// streaming / evict-first path (ld.global.cs): every byte is touched once.
// The grid is persistent (a multiple of the SM count, from the occupancy
// calculator) and strides over units.
//
// pack / unpack: one thread per unit transposes 32 elements in registers
// (bfp_layout.cuh); the plane side of every access is coalesced, the element
// side is a 32..128-B contiguous chunk per thread (vector loads).
#pragma once
#if !defined(__CUDACC_RTC__)
#include <cuda_runtime.h>

#include <algorithm>
#endif

#include "bfp_circuits.cuh"
#include "bfp_layout.cuh"

namespace bfpg {

enum Op { OP_ADD = 0, OP_SUB = 1, OP_MUL = 2, OP_DIV = 3, OP_MUL_ADD = 4 };

constexpr int kThreads = 128;

__device__ __forceinline__ w32 ld_stream(const w32* p) { return __ldcs(p); }

// Programmatic dependent launch: every kernel waits for the previous grid to
// complete -- memory included -- before its first global access (so
// stream-ordered dependent calls remain correct), and each CTA releases the
// next kernel after its last unit, so the successor's CTAs fill SMs as ours
// retire.  (Releasing at entry measured worse on mixed multi-kernel steps:
// C4 -9%; the late release keeps the C2 gain, +6%.)  No-ops when the launch
// did not enable PDL.
#ifndef BFP_PDL_EARLY
#define BFP_PDL_EARLY 0
#endif
__device__ __forceinline__ void pdl_enter() {
#if BFP_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
// Late release: called by each CTA after its last unit (no-op when the
// release already happened at entry).
__device__ __forceinline__ void pdl_release() {
#if !BFP_PDL_EARLY
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}
// The same release issued from inside a grid-stride loop, by each thread
// after the stores of its last unit.  A release after the
// loop makes ptxas re-materialise the memory descriptor into a fresh uniform
// register pair (R2UR) for every LDG/STG of the body -- 72 extra ALU-pipe
// instructions per unit on 1/5/10 mul, ~11% of a logic-bound kernel; issued
// under a predicate inside the loop it does not.  Dependents only start once
// every thread has released or exited, and their griddepcontrol.wait still
// waits for this grid's completion, so the timing is all that changes.
__device__ __forceinline__ void pdl_release_if(bool last) {
#if !BFP_PDL_EARLY
  if (last) asm volatile("griddepcontrol.launch_dependents;");
#endif
}
__device__ __forceinline__ void st_stream(w32* p, w32 v) { __stcs(p, v); }

// Operands of one unit: NIN inputs x N planes, loaded with the streaming path.
template <int N, int NIN>
struct Operands {
  w32 v[NIN][N];
  __device__ __forceinline__ void load(const w32* __restrict__ x, const w32* __restrict__ y,
                                       const w32* __restrict__ c, size_t base) {
    BFP_UNROLL for (int j = 0; j < N; ++j) {
      v[0][j] = ld_stream(x + base + j * 32);
      v[1][j] = ld_stream(y + base + j * 32);
      if constexpr (NIN == 3) v[2][j] = ld_stream(c + base + j * 32);
    }
  }
};

template <class F, int OP>
__device__ __forceinline__ void eval_unit(const w32* X, const w32* Y, const w32* Cc, w32* Z) {
  if constexpr (Gen<F, OP>::ok) {
    Gen<F, OP>::run(X, Y, Cc, Z);  // LOP3-mapped cover of the same network
  } else if constexpr (OP == OP_ADD) {
    add_w<F, false>(X, Y, Z);
  } else if constexpr (OP == OP_SUB) {
    add_w<F, true>(X, Y, Z);
  } else if constexpr (OP == OP_MUL) {
    mul_w<F>(X, Y, Z);
  } else if constexpr (OP == OP_DIV) {
    div_w<F>(X, Y, Z);
  } else {
    mul_add_w<F>(X, Y, Cc, Z);
  }
}

// mul_add with a fast-domain cover (Gen<F, 5>, bfp_circuits.cuh
// mul_add_fast_domain): every lane evaluates the domain predicate of its unit
// (~14 LOP3) and the warp votes, so all 32 lanes run the SAME cover -- the
// fast one only when all 1024 elements of the block are inside the domain.
// BFP_GENERAL_NETWORK (flags bit 1) forces the general cover.  All 32 lanes of
// a warp are in the loop together (units is a multiple of 32 and a warp owns
// 32 consecutive units), so the full-mask vote is safe.
constexpr int OP_MUL_ADD_FAST = 5;
// Formats without generated covers (the NVRTC backend's runtime formats) use
// the fast-domain TEMPLATE the same way.
template <class F, int OP>
constexpr bool has_fast_cover() {
  if constexpr (OP == OP_MUL_ADD)
    return Gen<F, OP_MUL_ADD_FAST>::ok || (!Gen<F, OP_MUL_ADD>::ok && mul_add_fast_ok<F>());
  return false;
}
template <class F, int OP>
__device__ __forceinline__ void eval_unit_dyn(const w32* X, const w32* Y, const w32* Cc, w32* Z,
                                              unsigned flags) {
  if constexpr (has_fast_cover<F, OP>()) {
    const bool in_domain = mul_add_fast_domain<F>(X, Y, Cc) == ONES;
    if (__all_sync(0xffffffffu, in_domain) && !(flags & 2u)) {
      if constexpr (Gen<F, OP_MUL_ADD_FAST>::ok)
        Gen<F, OP_MUL_ADD_FAST>::run(X, Y, Cc, Z);
      else
        mul_add_fast_w<F>(X, Y, Cc, Z);
      return;
    }
  }
  eval_unit<F, OP>(X, Y, Cc, Z);
}

// How many blocks of a mul_add call run the fast-domain cover: the same
// predicate on the same planes and the same warp vote as k_arith (only the
// exponent planes are read).  Introspection for callers, tests and the bench.
template <class F>
__global__ void __launch_bounds__(kThreads) k_fast_blocks(const w32* __restrict__ a,
                                                          const w32* __restrict__ b,
                                                          const w32* __restrict__ c, size_t units,
                                                          unsigned long long* __restrict__ count) {
  constexpr int N = F::N, S = F::S, E = F::E;
  const size_t stride = size_t(gridDim.x) * kThreads;
  unsigned long long mine = 0;
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    bool in_domain = false;
    if constexpr (has_fast_cover<F, OP_MUL_ADD>()) {
      w32 A[N], B[N], Cc[N];
      BFP_UNROLL for (int j = S; j < S + E; ++j) {
        A[j] = a[base + j * 32];
        B[j] = b[base + j * 32];
        Cc[j] = c[base + j * 32];
      }
      in_domain = mul_add_fast_domain<F>(A, B, Cc) == ONES;
    }
    if (__all_sync(0xffffffffu, in_domain) && (threadIdx.x & 31) == 0) ++mine;
  }
  if (mine) atomicAdd(count, mine);
}

// One thread per unit, grid-stride.  (A register double-buffered variant --
// next unit's loads issued before the current network -- measured slower on
// the B200: the extra registers cost more occupancy than the overlap gained.)
#ifndef BFP_ARITH_MINB
#define BFP_ARITH_MINB 1
#endif
// Minimum resident CTAs per SM asked of ptxas.  Mid-size logic-bound networks
// (mul / div of 300-800 LOP3 per word: 1/5/7, 1/5/10, 1/6/9, 1/8/7) come out
// at 90-100 registers unconstrained (5 CTAs/SM); capping them for 6 CTAs
// costs no spills and measured +10% on 1/8/7 mul, +2-5% on 1/5/10 mul.  Small
// networks are HBM-bound (the cap measured -2..-3% there).  The 1/8/15 mul
// (~1000 LOP3 per word, 137 registers uncapped = 3 CTAs/SM) capped for 4
// CTAs/SM (115 registers, no spills) measured +4% in two repeated A/Bs
// (profiles/r01_ab_minb_wide.txt).  mul_add capped for 5 CTAs/SM (1/6/9:
// 91 registers instead of 121, no spills (with the second, fast-domain cover in
// the kernel the 1/5/10 chain spills 12-20 B in three of its modes), +9 LOP3 of
// ptxas re-materialisation) measured +1.0% on C5 in a 4-round interleaved
// A/B (profiles/r02_ab_muladd_minb5.txt: 639.6 vs 633.2 Gelem/s, every
// round ahead); 6 spills.
#ifndef BFP_MID_MINB
#define BFP_MID_MINB 6
#endif
#ifndef BFP_WIDE_MINB
#define BFP_WIDE_MINB 4
#endif
#ifndef BFP_MULADD_MINB
#define BFP_MULADD_MINB 5
#endif
template <class F, int OP>
constexpr int arith_minb() {
  if constexpr (Gen<F, OP>::ok) {
    constexpr int l = Gen<F, OP>::luts;
    if ((OP == OP_MUL || OP == OP_DIV) && l >= 300 && l <= 800) return BFP_MID_MINB;
    if ((OP == OP_MUL || OP == OP_DIV) && l > 800 && l <= 1100) return BFP_WIDE_MINB;
    if (OP == OP_MUL_ADD && l >= 300 && l <= 1000) return BFP_MULADD_MINB;
  }
  return BFP_ARITH_MINB;
}

// L2 prefetch of the warp's NEXT block for the logic-bound networks: their
// units are long, so the next unit's loads then start from L2 instead of HBM
// and the unit-start stall shortens.  Each lane prefetches one or two of the
// block's NIN x N plane lines (prefetch.global.L2, per-thread addresses fixed
// before the loop: one 64-bit add per line per unit).  BFP_PREFETCH: 0 off,
// 1 networks of >= 300 LOP3 per word, 2 every arithmetic kernel.  Off by
// default: an interleaved A/B (profiles/r02_ab_prefetch.txt) showed no gain on
// the logic-bound networks (C5 mul_add 591 vs 602 Gelem/s without, 1/8/15
// mul 444 vs 456) for +10 ALU-pipe instructions per unit.
#ifndef BFP_PREFETCH
#define BFP_PREFETCH 0
#endif
__device__ __forceinline__ void prefetch_line_l2(const void* p) {
  asm volatile("prefetch.global.L2 [%0];" ::"l"(p));
}
template <class F, int OP>
constexpr bool arith_prefetch() {
  if constexpr (Gen<F, OP>::ok) return BFP_PREFETCH == 2 || (BFP_PREFETCH == 1 && Gen<F, OP>::luts >= 300);
  return BFP_PREFETCH == 2;
}

template <class F, int OP>
__global__ void __launch_bounds__(kThreads, arith_minb<F, OP>()) k_arith(const w32* __restrict__ x,
                                                    const w32* __restrict__ y,
                                                    const w32* __restrict__ c,
                                                    w32* __restrict__ z, size_t units,
                                                    unsigned flags) {
  // BFP_INPUTS_READY (flags bit 0): the caller guarantees that no work still
  // running on the stream writes x / y / c, so each thread issues its first
  // unit's loads before griddepcontrol.wait -- they overlap the previous
  // kernel's tail -- and waits before its first store (no WAR / WAW hazard).
  bool waited = !(flags & 1u);
  if (waited) pdl_enter();
  constexpr int N = F::N;
  constexpr int NIN = OP == OP_MUL_ADD ? 3 : 2;
  const size_t stride = size_t(gridDim.x) * kThreads;
  // this lane's prefetch lines l = lane, lane + 32 of a block (operand l / N,
  // plane l % N; taken modulo the block's NIN x N lines, so every pointer is
  // valid and a few lines are simply prefetched twice), as pointers into block 0
  constexpr int NPF = NIN * N > 32 ? 2 : 1;
  const w32* pf[NPF];
  BFP_UNROLL for (int k = 0; k < NPF; ++k) {
    const unsigned l = ((threadIdx.x & 31) + 32 * k) % unsigned(NIN * N);
    pf[k] = (l < N ? x : (l < 2 * N ? y : c)) + (l % N) * 32;
  }
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    Operands<N, NIN> cur;
    cur.load(x, y, c, base);
    if (!waited) {
      asm volatile("griddepcontrol.wait;" ::: "memory");
      waited = true;
    }
    if constexpr (arith_prefetch<F, OP>()) {
      const size_t un = u + stride;
      if (un < units) {
        const size_t nb = (un >> 5) * (size_t(N) * 32);
        BFP_UNROLL for (int k = 0; k < NPF; ++k) prefetch_line_l2(pf[k] + nb);
      }
    }
    // register-capped networks: releasing before the network keeps the
    // loop-carried values out of local memory (ptxas spilled 20-24 B of the
    // 1/5/10 and 1/6/9 mul loops with the release after the stores)
    if constexpr (arith_minb<F, OP>() > 1) pdl_release_if(u + stride >= units);
    w32 Z[N];
    eval_unit_dyn<F, OP>(cur.v[0], cur.v[1], cur.v[NIN - 1], Z, flags);
    BFP_UNROLL for (int j = 0; j < N; ++j) st_stream(z + base + j * 32, Z[j]);
    if constexpr (arith_minb<F, OP>() <= 1) pdl_release_if(u + stride >= units);
  }
}

// ---------------------------------------------- bulk-copy pipelined variant
// Each warp streams its blocks through a STAGES-deep ring in shared memory:
// one lane issues cp.async.bulk (global -> shared, completion counted on an
// mbarrier with expect_tx) for the NIN operand tiles of a block -- a block's
// N planes are contiguous, N x 128 B per operand -- STAGES blocks ahead; all
// lanes wait on the stage's mbarrier phase, read their plane words with
// conflict-free LDS.32, hand the stage back, evaluate the network and store
// the result planes with coalesced STG.  Loads stay in flight during the
// network instead of alternating with it.
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_addr(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_addr(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}

#ifndef BFP_BULK_BUDGET
#define BFP_BULK_BUDGET (16 * 1024)  // ring bytes per warp
#endif
template <int N, int NIN>
constexpr int bulk_stages() {
  constexpr int stage_bytes = NIN * N * 128;
  constexpr int s = (BFP_BULK_BUDGET) / stage_bytes;
  return s < 2 ? 2 : (s > 4 ? 4 : s);
}

template <class F, int OP>
__global__ void __launch_bounds__(kThreads) k_arith_bulk(const w32* __restrict__ x,
                                                         const w32* __restrict__ y,
                                                         const w32* __restrict__ c,
                                                         w32* __restrict__ z, size_t nblocks) {
  constexpr int N = F::N;
  constexpr int NIN = OP == OP_MUL_ADD ? 3 : 2;
  constexpr int ST = bulk_stages<N, NIN>();
  constexpr int TW = N * 32;  // words per operand tile
  extern __shared__ __align__(128) w32 dsm[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  w32* ring = dsm + wib * ST * NIN * TW;
  uint64_t* bars = reinterpret_cast<uint64_t*>(dsm + (kThreads / 32) * ST * NIN * TW) + wib * ST;
  if (lane == 0) {
    BFP_UNROLL for (int s = 0; s < ST; ++s) mbar_init(bars + s, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  pdl_enter();
  const size_t tw = size_t(gridDim.x) * (kThreads / 32);
  const size_t gw = size_t(blockIdx.x) * (kThreads / 32) + wib;
  const w32* src[3] = {x, y, c};
  auto issue = [&](int s, size_t b) {
    mbar_expect_tx(bars + s, NIN * TW * 4);
    BFP_UNROLL for (int a = 0; a < NIN; ++a)
      bulk_g2s(ring + (s * NIN + a) * TW, src[a] + b * TW, TW * 4, bars + s);
  };
  if (lane == 0) {
    BFP_UNROLL for (int s = 0; s < ST; ++s) {
      const size_t b = gw + size_t(s) * tw;
      if (b < nblocks) issue(s, b);
    }
  }
  int s = 0;
  uint32_t phase = 0;
  for (size_t b = gw; b < nblocks; b += tw) {
    mbar_wait(bars + s, phase);
    const w32* rs = ring + s * (NIN * TW) + lane;  // this stage, this lane's word column
    w32 ops[NIN][N];
    BFP_UNROLL for (int a = 0; a < NIN; ++a)
      BFP_UNROLL for (int j = 0; j < N; ++j) ops[a][j] = rs[a * TW + j * 32];
    __syncwarp();
    if (lane == 0) {
      const size_t bn = b + size_t(ST) * tw;
      if (bn < nblocks) issue(s, bn);
    }
    if (++s == ST) {
      s = 0;
      phase ^= 1u;
    }
    w32 Z[N];
    eval_unit_dyn<F, OP>(ops[0], ops[1], ops[NIN - 1], Z, 0u);  // the warp is converged here
    w32* zb = z + b * size_t(TW) + lane;
    BFP_UNROLL for (int j = 0; j < N; ++j) st_stream(zb + j * 32, Z[j]);
    pdl_release_if(b + tw >= nblocks);  // in-loop: see pdl_release_if (no per-access R2UR)
  }
}

// Logic-bound networks (LOP3 per byte of HBM traffic above the B200's
// ~2.9 LOP3/byte balance point, with margin) take the bulk-copy pipeline;
// HBM-bound ones keep the plain loop (measured: the ring's shared memory costs
// them occupancy, and 1-KB bulk tiles underuse the copy engine).
template <class F, int OP>
constexpr bool prefer_bulk() {
  if constexpr (Gen<F, OP>::ok) {
    constexpr int NIN = OP == OP_MUL_ADD ? 3 : 2;
    constexpr double lop3_per_elem = Gen<F, OP>::luts / 32.0;
    constexpr double bytes_per_elem = (NIN + 1) * F::N / 8.0;
    return lop3_per_elem / bytes_per_elem > 2.2;
  } else {
    return false;
  }
}

template <class F, int OP>
constexpr size_t bulk_smem_bytes() {
  constexpr int NIN = OP == OP_MUL_ADD ? 3 : 2;
  return size_t(kThreads / 32) * bulk_stages<F::N, NIN>() * (NIN * F::N * 128 + 8);
}

// ------------------------------------------------------------------ pack
// Loads the 32 encodings of unit u (element width EB bytes) into w32 words,
// zero beyond n.  Fast path: 16-B vector loads when the unit is complete.
template <int EB>
__device__ __forceinline__ void load_unit(const uint8_t* __restrict__ enc, size_t u, size_t n,
                                          bool aligned, w32* L) {
  constexpr int WORDS = 32 * EB / 4;
  const size_t e0 = u * 32;
  if (aligned && e0 + 32 <= n) {
    const uint4* p = reinterpret_cast<const uint4*>(enc + e0 * EB);
    BFP_UNROLL for (int i = 0; i < WORDS / 4; ++i) {
      const uint4 q = __ldcs(p + i);
      L[4 * i] = q.x;
      L[4 * i + 1] = q.y;
      L[4 * i + 2] = q.z;
      L[4 * i + 3] = q.w;
    }
  } else {
    BFP_UNROLL for (int i = 0; i < WORDS; ++i) L[i] = 0;
    const size_t nb = (n > e0) ? ((n - e0 < 32 ? n - e0 : 32) * EB) : 0;
    for (size_t b = 0; b < nb; ++b) L[b >> 2] |= w32(enc[e0 * EB + b]) << (8 * (b & 3));
  }
}

template <int EB>
__device__ __forceinline__ void store_unit(uint8_t* __restrict__ enc, size_t u, size_t n,
                                           bool aligned, const w32* L) {
  constexpr int WORDS = 32 * EB / 4;
  const size_t e0 = u * 32;
  if (e0 >= n) return;
  if (aligned && e0 + 32 <= n) {
    uint4* p = reinterpret_cast<uint4*>(enc + e0 * EB);
    BFP_UNROLL for (int i = 0; i < WORDS / 4; ++i)
      __stcs(p + i, make_uint4(L[4 * i], L[4 * i + 1], L[4 * i + 2], L[4 * i + 3]));
  } else {
    const size_t nb = (n - e0 < 32 ? n - e0 : 32) * EB;
    for (size_t b = 0; b < nb; ++b) enc[e0 * EB + b] = uint8_t(L[b >> 2] >> (8 * (b & 3)));
  }
}

// Warp-cooperative tile through shared memory: lane t owns row t (its
// unit's 32 elements = CH 16-byte chunks); global memory sees the tile
// row-major, so each warp instruction moves 512 contiguous bytes.  Chunks
// are XOR-swizzled by row so the row-wise and the flat accesses are both
// (nearly) bank-conflict free.  Requires the whole warp active.
template <int CH>
__device__ __forceinline__ int tile_off(int row, int chunk) {
  if constexpr ((CH & (CH - 1)) == 0) return row * (CH * 4) + ((chunk ^ (row & (CH - 1))) << 2);
  else return row * (CH * 4) + (((chunk + row) % CH) << 2);
}

template <int CH>
__device__ __forceinline__ void tile_store_rows(w32* tile, const w32* V, int lane) {
  BFP_UNROLL for (int c = 0; c < CH; ++c)
    *reinterpret_cast<uint4*>(tile + tile_off<CH>(lane, c)) =
        make_uint4(V[4 * c], V[4 * c + 1], V[4 * c + 2], V[4 * c + 3]);
}

template <int CH>
__device__ __forceinline__ void tile_load_rows(const w32* tile, w32* V, int lane) {
  BFP_UNROLL for (int c = 0; c < CH; ++c) {
    const uint4 q = *reinterpret_cast<const uint4*>(tile + tile_off<CH>(lane, c));
    V[4 * c] = q.x;
    V[4 * c + 1] = q.y;
    V[4 * c + 2] = q.z;
    V[4 * c + 3] = q.w;
  }
}

// global (32 * CH * 4 contiguous words at g) <-> tile, flat order
template <int CH>
__device__ __forceinline__ void tile_from_global(w32* tile, const w32* __restrict__ g, int lane) {
  BFP_UNROLL for (int i = 0; i < CH; ++i) {
    const int flat = i * 128 + lane * 4;  // word index in the tile
    const uint4 q = __ldcs(reinterpret_cast<const uint4*>(g + flat));
    *reinterpret_cast<uint4*>(tile + tile_off<CH>(flat / (CH * 4), (flat % (CH * 4)) >> 2)) = q;
  }
}

template <int CH>
__device__ __forceinline__ void tile_to_global(const w32* tile, w32* __restrict__ g, int lane) {
  BFP_UNROLL for (int i = 0; i < CH; ++i) {
    const int flat = i * 128 + lane * 4;
    const uint4 q =
        *reinterpret_cast<const uint4*>(tile + tile_off<CH>(flat / (CH * 4), (flat % (CH * 4)) >> 2));
    __stcs(reinterpret_cast<uint4*>(g + flat), q);
  }
}

// Element side of one warp's 1024 elements (EB bytes each): coalesced via the
// tile when the warp's range is complete and 16-B aligned; otherwise each lane
// moves its own unit's bytes between global memory and its tile row one byte
// at a time (zero past n).  Either way the registers are filled from / drained
// to the tile with static indices only -- a dynamically indexed register
// array would be demoted to local memory for the fast path as well.
template <int CH>
__device__ __forceinline__ w32* tile_word(w32* tile, int row, int word) {
  return tile + tile_off<CH>(row, word >> 2) + (word & 3);
}

template <int EB>
__device__ __forceinline__ void warp_load_elems(const uint8_t* __restrict__ src, size_t u, size_t n,
                                                bool aligned, w32* tile, int lane, w32* L) {
  constexpr int CH = 2 * EB;
  const size_t e0w = (u - lane) * 32;
  if (aligned && e0w + 1024 <= n) {
    tile_from_global<CH>(tile, reinterpret_cast<const w32*>(src + e0w * EB), lane);
  } else {
    const size_t e0 = u * 32;
    const size_t nb = (n > e0) ? ((n - e0 < 32 ? n - e0 : 32) * EB) : 0;
    for (int w = 0; w < 8 * EB; ++w) {
      w32 v = 0;
      for (int t = 0; t < 4; ++t) {
        const size_t b = size_t(4 * w + t);
        if (b < nb) v |= w32(src[e0 * EB + b]) << (8 * t);
      }
      *tile_word<CH>(tile, lane, w) = v;
    }
  }
  __syncwarp();
  tile_load_rows<CH>(tile, L, lane);
  __syncwarp();
}

template <int EB>
__device__ __forceinline__ void warp_store_elems(uint8_t* __restrict__ dst, size_t u, size_t n,
                                                 bool aligned, w32* tile, int lane, const w32* L) {
  constexpr int CH = 2 * EB;
  const size_t e0w = (u - lane) * 32;
  tile_store_rows<CH>(tile, L, lane);
  __syncwarp();
  if (aligned && e0w + 1024 <= n) {
    tile_to_global<CH>(tile, reinterpret_cast<w32*>(dst + e0w * EB), lane);
  } else {
    const size_t e0 = u * 32;
    const size_t nb = (n > e0) ? ((n - e0 < 32 ? n - e0 : 32) * EB) : 0;
    for (size_t b = 0; b < nb; ++b)
      dst[e0 * EB + b] = uint8_t(*tile_word<CH>(tile, lane, int(b >> 2)) >> (8 * (b & 3)));
  }
  __syncwarp();
}

// Raw encodings / .bfpraw records (EB bytes each: 1, 2, 4, 8 = the device
// encoding widths; 3, 5, 6, 7 = .bfpraw strides) -> planes.  Every unit of
// every block is written; elements >= n are zero (pack.hpp:50).
template <int N, int EB>
__global__ void __launch_bounds__(kThreads) k_pack_enc(const uint8_t* __restrict__ enc,
                                                       w32* __restrict__ planes, size_t n,
                                                       size_t units, bool aligned) {
  pdl_enter();
  constexpr int PW = EB > 4 ? 64 : 32;
  __shared__ __align__(16) w32 tiles[kThreads / 32][256 * EB];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {
    w32 L[8 * EB];
    warp_load_elems<EB>(enc, u, n, aligned, tile, lane, L);
    w32 P[PW];
    elems_to_planes<EB>(L, P);
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    BFP_UNROLL for (int j = 0; j < N; ++j) st_stream(planes + base + j * 32, P[j]);
    pdl_release_if(u + stride >= units);
  }
}

template <int N, int EB>
__global__ void __launch_bounds__(kThreads) k_unpack_enc(const w32* __restrict__ planes,
                                                         uint8_t* __restrict__ enc, size_t n,
                                                         size_t units, bool aligned) {
  pdl_enter();
  constexpr int PW = EB > 4 ? 64 : 32;
  __shared__ __align__(16) w32 tiles[kThreads / 32][256 * EB];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  const size_t wunits = (units + 31) & ~size_t(31);  // whole warps (planes exist)
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < wunits; u += stride) {
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    w32 P[PW];
    BFP_UNROLL for (int j = 0; j < PW; ++j) P[j] = (j < N) ? ld_stream(planes + base + j * 32) : 0u;
    w32 L[8 * EB];
    planes_to_elems<EB>(P, L);
    warp_store_elems<EB>(enc, u, n, aligned, tile, lane, L);
    pdl_release_if(u + stride >= wunits);
  }
}

// 32 float32 bit patterns of one unit -> the unit's N plane words (encode_scalar
// semantics).  Hardware cvt (binary16 / bfloat16) where it coincides with the
// reference converter, else the branch-free per-element encoder; then the
// register transpose.
template <class F>
__device__ __forceinline__ void floats_to_planes(w32* V, w32* P) {
  constexpr int N = F::N;
  constexpr int HW = HwCodec<F>::kind;
  if constexpr (HW != 0) {
    w32 L[16];
    BFP_UNROLL for (int q = 0; q < 16; ++q)
      L[q] = hw_cvt2<HW, F::RN>(__uint_as_float(V[2 * q]), __uint_as_float(V[2 * q + 1]));
    enc16_to_planes(L, P);
    canon_nan_planes<F>(P);
    if constexpr (F::FTZ) {  // subnormal results -> signed zero: clear their fraction planes
      w32 h = 0;
      BFP_UNROLL for (int i = 0; i < F::E; ++i) h |= P[F::S + i];
      BFP_UNROLL for (int j = 0; j < F::S; ++j) P[j] &= h;
    }
  } else {
    BFP_UNROLL for (int k = 0; k < 32; ++k) V[k] = encode_f32_fast<F>(V[k]);
    if constexpr (N <= 8) {
      w32 L[8];
      BFP_UNROLL for (int q = 0; q < 8; ++q)
        L[q] = V[4 * q] | (V[4 * q + 1] << 8) | (V[4 * q + 2] << 16) | (V[4 * q + 3] << 24);
      enc8_to_planes(L, P);
    } else if constexpr (N <= 16) {
      w32 L[16];
      BFP_UNROLL for (int q = 0; q < 16; ++q) L[q] = V[2 * q] | (V[2 * q + 1] << 16);
      enc16_to_planes(L, P);
    } else {
      BFP_UNROLL for (int i = 0; i < 32; ++i) P[i] = V[i];
      enc32_to_planes(P);
    }
  }
}

// The unit's N plane words -> 32 float32 bit patterns ((float)decode_scalar).
// P is clobbered (32 words, rows >= N must be zero).
template <class F>
__device__ __forceinline__ void planes_to_floats(w32* P, w32* V) {
  constexpr int N = F::N;
  constexpr int HW = HwCodec<F>::kind;
  if constexpr (HW != 0) {
    canon_nan_planes<F>(P);  // 0x7e00 / 0x7fc0 widen to 0x7fc00000
    w32 L[16];
    planes_to_enc16(P, L);
    BFP_UNROLL for (int q = 0; q < 16; ++q) {
      V[2 * q] = hw_widen<HW>(L[q] & 0xffffu);
      V[2 * q + 1] = hw_widen<HW>(L[q] >> 16);
    }
  } else {
    if constexpr (N <= 8) {
      w32 L[8];
      planes_to_enc8(P, L);
      BFP_UNROLL for (int k = 0; k < 32; ++k) V[k] = (L[k >> 2] >> (8 * (k & 3))) & 0xffu;
    } else if constexpr (N <= 16) {
      w32 L[16];
      planes_to_enc16(P, L);
      BFP_UNROLL for (int k = 0; k < 32; ++k) V[k] = (L[k >> 1] >> (16 * (k & 1))) & 0xffffu;
    } else {
      planes_to_enc32(P);
      BFP_UNROLL for (int k = 0; k < 32; ++k) V[k] = P[k];
    }
    BFP_UNROLL for (int k = 0; k < 32; ++k) V[k] = decode_f32_fast<F>(V[k]);
  }
}

// float32 -> encode_scalar -> planes.
template <class F>
__global__ void __launch_bounds__(kThreads) k_pack_f32(const float* __restrict__ in,
                                                       w32* __restrict__ planes, size_t n,
                                                       size_t units, bool aligned) {
  pdl_enter();
  constexpr int N = F::N;
  __shared__ __align__(16) w32 tiles[kThreads / 32][1024];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  const uint8_t* inb = reinterpret_cast<const uint8_t*>(in);
  // units is a multiple of 32 (whole blocks), so warps stay converged
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {
    w32 V[32];
    warp_load_elems<4>(inb, u, n, aligned, tile, lane, V);  // zero past n -> +0 -> 0
    w32 P[32];
    floats_to_planes<F>(V, P);
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    BFP_UNROLL for (int j = 0; j < N; ++j) st_stream(planes + base + j * 32, P[j]);
    pdl_release_if(u + stride >= units);
  }
}

// planes -> decode_scalar -> float32.
template <class F>
__global__ void __launch_bounds__(kThreads) k_unpack_f32(const w32* __restrict__ planes,
                                                         float* __restrict__ out, size_t n,
                                                         size_t units, bool aligned) {
  pdl_enter();
  constexpr int N = F::N;
  __shared__ __align__(16) w32 tiles[kThreads / 32][1024];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  uint8_t* outb = reinterpret_cast<uint8_t*>(out);
  const size_t wunits = (units + 31) & ~size_t(31);  // whole warps (planes exist)
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < wunits; u += stride) {
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    w32 P[32];
    BFP_UNROLL for (int j = 0; j < 32; ++j) P[j] = (j < N) ? ld_stream(planes + base + j * 32) : 0u;
    w32 V[32];
    planes_to_floats<F>(P, V);
    warp_store_elems<4>(outb, u, n, aligned, tile, lane, V);
    pdl_release_if(u + stride >= wunits);
  }
}

// binary64 -> encode_scalar -> planes (format.hpp:125-188, the reference
// converter's own input type), any legal format.
template <class F>
__global__ void __launch_bounds__(kThreads) k_pack_f64(const double* __restrict__ in,
                                                       w32* __restrict__ planes, size_t n,
                                                       size_t units, bool aligned) {
  pdl_enter();
  constexpr int N = F::N;
  __shared__ __align__(16) w32 tiles[kThreads / 32][2048];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  const uint8_t* inb = reinterpret_cast<const uint8_t*>(in);
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {
    w32 L[64];
    warp_load_elems<8>(inb, u, n, aligned, tile, lane, L);  // zero past n -> +0 -> 0
    BFP_UNROLL for (int k = 0; k < 32; ++k) {
      const uint64_t e = encode_f64<F>(uint64_t(L[2 * k]) | (uint64_t(L[2 * k + 1]) << 32));
      L[2 * k] = w32(e);
      L[2 * k + 1] = w32(e >> 32);
    }
    w32 P[64];
    elems_to_planes<8>(L, P);
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    BFP_UNROLL for (int j = 0; j < N; ++j) st_stream(planes + base + j * 32, P[j]);
    pdl_release_if(u + stride >= units);
  }
}

// planes -> decode_scalar -> binary64 (exact).
template <class F>
__global__ void __launch_bounds__(kThreads) k_unpack_f64(const w32* __restrict__ planes,
                                                         double* __restrict__ out, size_t n,
                                                         size_t units, bool aligned) {
  pdl_enter();
  constexpr int N = F::N;
  __shared__ __align__(16) w32 tiles[kThreads / 32][2048];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  uint8_t* outb = reinterpret_cast<uint8_t*>(out);
  const size_t wunits = (units + 31) & ~size_t(31);
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < wunits; u += stride) {
    const size_t base = (u >> 5) * (size_t(N) * 32) + (u & 31);
    w32 P[64];
    BFP_UNROLL for (int j = 0; j < 64; ++j) P[j] = (j < N) ? ld_stream(planes + base + j * 32) : 0u;
    w32 L[64];
    planes_to_elems<8>(P, L);
    BFP_UNROLL for (int k = 0; k < 32; ++k) {
      const uint64_t d = decode_f64<F>(uint64_t(L[2 * k]) | (uint64_t(L[2 * k + 1]) << 32));
      L[2 * k] = w32(d);
      L[2 * k + 1] = w32(d >> 32);
    }
    warp_store_elems<8>(outb, u, n, aligned, tile, lane, L);
    pdl_release_if(u + stride >= wunits);
  }
}

// Fused float32-in / float32-out arithmetic: the
// operands are converted to planes in registers, the network runs, the
// result is converted back -- the bitslice intermediate never reaches HBM
// (4 B/elem per operand in, 4 B/elem out).  Equals
// unpack_f32(op(pack_f32(x), pack_f32(y)[, pack_f32(c)])).
template <class F, int OP>
__global__ void __launch_bounds__(kThreads) k_arith_f32(const float* __restrict__ x,
                                                        const float* __restrict__ y,
                                                        const float* __restrict__ c,
                                                        float* __restrict__ z, size_t n,
                                                        size_t units, bool aligned) {
  pdl_enter();
  constexpr int N = F::N;
  constexpr int NIN = OP == OP_MUL_ADD ? 3 : 2;
  __shared__ __align__(16) w32 tiles[kThreads / 32][1024];
  const int lane = threadIdx.x & 31;
  w32* tile = tiles[threadIdx.x >> 5];
  const size_t stride = size_t(gridDim.x) * kThreads;
  const float* src[3] = {x, y, c};
  for (size_t u = size_t(blockIdx.x) * kThreads + threadIdx.x; u < units; u += stride) {
    w32 ops[NIN][N];
    BFP_UNROLL for (int a = 0; a < NIN; ++a) {
      w32 V[32], P[32];
      warp_load_elems<4>(reinterpret_cast<const uint8_t*>(src[a]), u, n, aligned, tile, lane, V);
      floats_to_planes<F>(V, P);
      BFP_UNROLL for (int j = 0; j < N; ++j) ops[a][j] = P[j];
    }
    w32 P[32];
    eval_unit<F, OP>(ops[0], ops[1], ops[NIN - 1], P);
    BFP_UNROLL for (int j = N; j < 32; ++j) P[j] = 0;
    w32 V[32];
    planes_to_floats<F>(P, V);
    warp_store_elems<4>(reinterpret_cast<uint8_t*>(z), u, n, aligned, tile, lane, V);
    pdl_release_if(u + stride >= units);
  }
}

// ------------------------------------------------------- launch + table
#if !defined(__CUDACC_RTC__)  // host-side launch code (not under NVRTC)
bool pdl_enabled();  // bfp_capi.cu: BFP_PDL environment switch (default on)

template <typename... KArgs, typename... Args>
inline cudaError_t launch(void (*k)(KArgs...), int grid, cudaStream_t st, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_smem(void (*k)(KArgs...), int grid, size_t smem, cudaStream_t st,
                               Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, k, static_cast<KArgs>(args)...);
}

int bulk_mode();   // bfp_capi.cu: BFP_BULK = 0 off (default) / 1 auto / 2 force
int grid_mult();   // bfp_capi.cu: BFP_GRID_MULT (default 4): CTA waves per grid

// Resident CTAs for a full wave of `kernel`: #SM x occupancy.
template <typename K>
inline int wave_ctas(K kernel, size_t smem = 0) {
  int dev = 0, sms = 0, occ = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, kThreads, smem);
  if (occ <= 0) occ = 1;
  return sms * occ;
}

// Grid: a whole number k <= grid_mult() (default 4) of resident waves
// (#SM x occupancy).  Oversubscription lets the CTA scheduler backfill SMs at
// the tail (+5-8% on large HBM-bound launches); k is the largest that still
// gives every thread >= 2 units (single-unit CTAs measured slower).  Whole
// waves only: a partial last wave (the old "need/2 CTAs" rule gave 1.38 waves
// at 2^24 elements) leaves most SMs idle while its CTAs run.
inline int grid_for(int wave, size_t units) {
  const size_t need = (units + kThreads - 1) / kThreads;
  if (need <= size_t(wave)) return int(need ? need : 1);
  size_t k = size_t(grid_mult());
  while (k > 1 && k * size_t(wave) * kThreads * 2 > units) --k;
  return int(k * size_t(wave));
}

// Per-format entry points: implemented by the compiled networks
// (FormatImpl<F>, instantiated in inst/fmt_E_S.cu) and by the NVRTC
// runtime-format backend (bfp_jit.cu) for every other legal format.
struct Impl {
  virtual ~Impl() = default;
  virtual cudaError_t arith(int op, const w32* x, const w32* y, const w32* c, w32* z,
                            size_t nblocks, cudaStream_t st, unsigned flags = 0) const = 0;
  virtual cudaError_t pack_enc(const void* enc, w32* planes, size_t n, cudaStream_t st) const = 0;
  virtual cudaError_t unpack_enc(const w32* planes, void* enc, size_t n, cudaStream_t st) const = 0;
  virtual cudaError_t pack_f32(const float* in, w32* planes, size_t n, cudaStream_t st) const = 0;
  virtual cudaError_t unpack_f32(const w32* planes, float* out, size_t n, cudaStream_t st) const = 0;
  // .bfpraw records (stride ceil(N/8) bytes; equal to pack_enc/unpack_enc when
  // the stride is the device encoding width 1/2/4/8)
  virtual cudaError_t pack_raw(const void* bytes, w32* planes, size_t n, cudaStream_t st) const = 0;
  virtual cudaError_t unpack_raw(const w32* planes, void* bytes, size_t n, cudaStream_t st) const = 0;
  // fused float32-in / float32-out arithmetic
  virtual cudaError_t arith_f32(int op, const float* x, const float* y, const float* c, float* z,
                                size_t n, cudaStream_t st) const = 0;
  // binary64 codec (encode_scalar / decode_scalar), any legal format
  virtual cudaError_t pack_f64(const double* in, w32* planes, size_t n, cudaStream_t st) const = 0;
  virtual cudaError_t unpack_f64(const w32* planes, double* out, size_t n, cudaStream_t st) const = 0;
  virtual const void* kernel(int id) const = 0;  // device function handle (attribute queries)
  virtual bool compiled() const { return true; }
  // blocks of a mul_add call that run the fast-domain cover (*d_count += them)
  virtual cudaError_t fast_blocks(const w32*, const w32*, const w32*, size_t, unsigned long long*,
                                  cudaStream_t) const {
    return cudaErrorNotSupported;
  }
};

template <class F>
struct FormatImpl {
  static constexpr int N = F::N;
  static constexpr int EB = N <= 8 ? 1 : (N <= 16 ? 2 : (N <= 32 ? 4 : 8));
  static constexpr int RAW = (N + 7) / 8;  // .bfpraw stride

  template <int OP>
  static cudaError_t launch_arith(const w32* x, const w32* y, const w32* c, w32* z, size_t units,
                                  cudaStream_t st, unsigned flags) {
    const int bulk = bulk_mode();  // 0 off, 1 auto (prefer_bulk), 2 force
    if (bulk == 2 || (bulk == 1 && prefer_bulk<F, OP>())) {
      auto kb = k_arith_bulk<F, OP>;
      constexpr size_t smem = bulk_smem_bytes<F, OP>();
      static const int wave_b = [&] {
        cudaFuncSetAttribute(kb, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        return wave_ctas(kb, smem);
      }();
      const size_t nblocks = units / 32;
      const size_t warps = (nblocks + 0);  // one block per warp-iteration
      const int grid = int(std::min<size_t>(size_t(wave_b), (warps + kThreads / 32 - 1) / (kThreads / 32)));
      return launch_smem(kb, grid > 0 ? grid : 1, smem, st, x, y, c, z, nblocks);
    }
    auto k = k_arith<F, OP>;
    static const int wave = wave_ctas(k);
    return launch(k, grid_for(wave, units), st, x, y, c, z, units, flags);
  }
  static cudaError_t arith(int op, const w32* x, const w32* y, const w32* c, w32* z,
                           size_t nblocks, cudaStream_t st, unsigned flags) {
    const size_t units = nblocks * 32;
    if (!units) return cudaSuccess;
    switch (op) {
      case OP_ADD: return launch_arith<OP_ADD>(x, y, c, z, units, st, flags);
      case OP_SUB: return launch_arith<OP_SUB>(x, y, c, z, units, st, flags);
      case OP_MUL: return launch_arith<OP_MUL>(x, y, c, z, units, st, flags);
      case OP_DIV: return launch_arith<OP_DIV>(x, y, c, z, units, st, flags);
      case OP_MUL_ADD: return launch_arith<OP_MUL_ADD>(x, y, c, z, units, st, flags);
      default: return cudaErrorInvalidValue;
    }
  }
  static const void* kernel(int op) {
    switch (op) {
      case OP_ADD: return reinterpret_cast<const void*>(k_arith<F, OP_ADD>);
      case OP_SUB: return reinterpret_cast<const void*>(k_arith<F, OP_SUB>);
      case OP_MUL: return reinterpret_cast<const void*>(k_arith<F, OP_MUL>);
      case OP_DIV: return reinterpret_cast<const void*>(k_arith<F, OP_DIV>);
      case OP_MUL_ADD: return reinterpret_cast<const void*>(k_arith<F, OP_MUL_ADD>);
      case 10: return reinterpret_cast<const void*>(k_pack_enc<N, EB>);
      case 11: return reinterpret_cast<const void*>(k_unpack_enc<N, EB>);
      case 12: return reinterpret_cast<const void*>(k_pack_f32<F>);
      case 13: return reinterpret_cast<const void*>(k_unpack_f32<F>);
      case 20: return reinterpret_cast<const void*>(k_arith_f32<F, OP_ADD>);
      case 22: return reinterpret_cast<const void*>(k_arith_f32<F, OP_MUL>);
      default: return nullptr;
    }
  }
  static size_t units_for(size_t n) { return ((n + 1023) / 1024) * 32; }
  static cudaError_t pack_enc(const void* enc, w32* planes, size_t n, cudaStream_t st) {
    const size_t units = units_for(n);
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(enc) & 15) == 0;
    auto k = k_pack_enc<N, EB>;
    static const int wave = wave_ctas(k);
    return launch(k, grid_for(wave, units), st, static_cast<const uint8_t*>(enc), planes, n,
                                                      units, al);
  }
  static cudaError_t unpack_enc(const w32* planes, void* enc, size_t n, cudaStream_t st) {
    const size_t units = (n + 31) / 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(enc) & 15) == 0;
    auto k = k_unpack_enc<N, EB>;
    static const int wave = wave_ctas(k);
    return launch(k, grid_for(wave, units), st, planes, static_cast<uint8_t*>(enc), n, units,
                                                      al);
  }
  static cudaError_t pack_f32(const float* in, w32* planes, size_t n, cudaStream_t st) {
    if constexpr (F::E > 8 || F::S > 23) {
      return cudaErrorNotSupported;
    } else {
      const size_t units = units_for(n);
      if (!units) return cudaSuccess;
      const bool al = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
      auto k = k_pack_f32<F>;
      static const int wave = wave_ctas(k);
      return launch(k, grid_for(wave, units), st, in, planes, n, units, al);
    }
  }
  static cudaError_t unpack_f32(const w32* planes, float* out, size_t n, cudaStream_t st) {
    if constexpr (F::E > 8 || F::S > 23) {
      return cudaErrorNotSupported;
    } else {
      const size_t units = (n + 31) / 32;
      if (!units) return cudaSuccess;
      const bool al = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
      auto k = k_unpack_f32<F>;
      static const int wave = wave_ctas(k);
      return launch(k, grid_for(wave, units), st, planes, out, n, units, al);
    }
  }
  static cudaError_t pack_raw(const void* bytes, w32* planes, size_t n, cudaStream_t st) {
    if constexpr (RAW == EB) {
      return pack_enc(bytes, planes, n, st);
    } else {
      const size_t units = units_for(n);
      if (!units) return cudaSuccess;
      const bool al = (reinterpret_cast<uintptr_t>(bytes) & 15) == 0;
      auto k = k_pack_enc<N, RAW>;
      static const int wave = wave_ctas(k);
      return launch(k, grid_for(wave, units), st, static_cast<const uint8_t*>(bytes), planes, n,
                    units, al);
    }
  }
  static cudaError_t unpack_raw(const w32* planes, void* bytes, size_t n, cudaStream_t st) {
    if constexpr (RAW == EB) {
      return unpack_enc(planes, bytes, n, st);
    } else {
      const size_t units = (n + 31) / 32;
      if (!units) return cudaSuccess;
      const bool al = (reinterpret_cast<uintptr_t>(bytes) & 15) == 0;
      auto k = k_unpack_enc<N, RAW>;
      static const int wave = wave_ctas(k);
      return launch(k, grid_for(wave, units), st, planes, static_cast<uint8_t*>(bytes), n, units,
                    al);
    }
  }
  static cudaError_t pack_f64(const double* in, w32* planes, size_t n, cudaStream_t st) {
    const size_t units = units_for(n);
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(in) & 15) == 0;
    auto k = k_pack_f64<F>;
    static const int wave = wave_ctas(k);
    return launch(k, grid_for(wave, units), st, in, planes, n, units, al);
  }
  static cudaError_t unpack_f64(const w32* planes, double* out, size_t n, cudaStream_t st) {
    const size_t units = (n + 31) / 32;
    if (!units) return cudaSuccess;
    const bool al = (reinterpret_cast<uintptr_t>(out) & 15) == 0;
    auto k = k_unpack_f64<F>;
    static const int wave = wave_ctas(k);
    return launch(k, grid_for(wave, units), st, planes, out, n, units, al);
  }
  template <int OP>
  static cudaError_t launch_arith_f32(const float* x, const float* y, const float* c, float* z,
                                     size_t n, cudaStream_t st) {
    const size_t units = units_for(n);
    if (!units) return cudaSuccess;
    const uintptr_t al_bits = reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(y) |
                              reinterpret_cast<uintptr_t>(z) |
                              (OP == OP_MUL_ADD ? reinterpret_cast<uintptr_t>(c) : 0);
    auto k = k_arith_f32<F, OP>;
    static const int wave = wave_ctas(k);
    return launch(k, grid_for(wave, units), st, x, y, c, z, n, units, (al_bits & 15) == 0);
  }
  static cudaError_t arith_f32(int op, const float* x, const float* y, const float* c, float* z,
                               size_t n, cudaStream_t st) {
    if constexpr (F::E > 8 || F::S > 23) {
      return cudaErrorNotSupported;
    } else {
      switch (op) {
        case OP_ADD: return launch_arith_f32<OP_ADD>(x, y, c, z, n, st);
        case OP_SUB: return launch_arith_f32<OP_SUB>(x, y, c, z, n, st);
        case OP_MUL: return launch_arith_f32<OP_MUL>(x, y, c, z, n, st);
        case OP_DIV: return launch_arith_f32<OP_DIV>(x, y, c, z, n, st);
        case OP_MUL_ADD: return launch_arith_f32<OP_MUL_ADD>(x, y, c, z, n, st);
        default: return cudaErrorInvalidValue;
      }
    }
  }
  struct Backend final : Impl {
    cudaError_t arith(int op, const w32* x, const w32* y, const w32* c, w32* z, size_t nb,
                      cudaStream_t st, unsigned flags) const override {
      return FormatImpl::arith(op, x, y, c, z, nb, st, flags);
    }
    cudaError_t pack_enc(const void* e, w32* p, size_t n, cudaStream_t st) const override {
      return FormatImpl::pack_enc(e, p, n, st);
    }
    cudaError_t unpack_enc(const w32* p, void* e, size_t n, cudaStream_t st) const override {
      return FormatImpl::unpack_enc(p, e, n, st);
    }
    cudaError_t pack_f32(const float* i, w32* p, size_t n, cudaStream_t st) const override {
      return FormatImpl::pack_f32(i, p, n, st);
    }
    cudaError_t unpack_f32(const w32* p, float* o, size_t n, cudaStream_t st) const override {
      return FormatImpl::unpack_f32(p, o, n, st);
    }
    cudaError_t pack_raw(const void* b, w32* p, size_t n, cudaStream_t st) const override {
      return FormatImpl::pack_raw(b, p, n, st);
    }
    cudaError_t unpack_raw(const w32* p, void* b, size_t n, cudaStream_t st) const override {
      return FormatImpl::unpack_raw(p, b, n, st);
    }
    cudaError_t arith_f32(int op, const float* x, const float* y, const float* c, float* z,
                          size_t n, cudaStream_t st) const override {
      return FormatImpl::arith_f32(op, x, y, c, z, n, st);
    }
    cudaError_t pack_f64(const double* i, w32* p, size_t n, cudaStream_t st) const override {
      return FormatImpl::pack_f64(i, p, n, st);
    }
    cudaError_t unpack_f64(const w32* p, double* o, size_t n, cudaStream_t st) const override {
      return FormatImpl::unpack_f64(p, o, n, st);
    }
    const void* kernel(int id) const override { return FormatImpl::kernel(id); }
    cudaError_t fast_blocks(const w32* a, const w32* b, const w32* c, size_t nb, unsigned long long* d_count,
                            cudaStream_t st) const override {
      const size_t units = nb * 32;
      if (!units) return cudaSuccess;
      auto k = k_fast_blocks<F>;
      static const int wave = wave_ctas(k);
      return launch(k, grid_for(wave, units), st, a, b, c, units, d_count);
    }
  };
  static const Impl* get() {
    static const Backend impl;
    return &impl;
  }
};

#endif  // !__CUDACC_RTC__

}  // namespace bfpg

#if !defined(__CUDACC_RTC__)
#define BFP_INSTANTIATE(E_, S_)                                                       \
  namespace bfpg {                                                                    \
  const Impl* impl_##E_##_##S_(int rn, int ftz) {                                     \
    if (rn && !ftz) return FormatImpl<Format<E_, S_, true, false>>::get();            \
    if (rn && ftz) return FormatImpl<Format<E_, S_, true, true>>::get();              \
    if (!rn && !ftz) return FormatImpl<Format<E_, S_, false, false>>::get();          \
    return FormatImpl<Format<E_, S_, false, true>>::get();                            \
  }                                                                                   \
  }
#endif

// bfp_circuits.cuh -- bitslice floating-point circuits for sm_100a.
//
// One uint32_t word ("w32") carries bit k of 32 elements: the device form of
// the reference's lane<W> (lane.hpp:28-117) at W = 32 per register.  Every
// function below is a fixed, data-independent network of AND/OR/XOR/NOT over
// such words; with the format a compile-time template (exponent bits E,
// fraction bits S, RN/RZ, gradual/FTZ) every loop unrolls and every constant
// folds, and ptxas maps the network onto 3-input LOP3 instructions.
//
// The networks are NOT a transcription of the reference circuits
// (circuits.hpp / arith.hpp).  They compute the same function -- correctly
// rounded IEEE-style add/sub/mul with the reference's conventions (canonical
// positive NaN format.hpp:49-52, +0 from cancellation arith.hpp:312-316,
// overflow to Inf/max-finite arith.hpp:143-146, FTZ after rounding with no
// input DAZ arith.hpp:135-141) -- with fewer gates:
//   * add: the alignment shift amount saturates instead of clearing the field,
//     the normaliser is budget-limited at the effective exponent of the larger
//     operand so subnormal sums land directly in place (no second shifter, no
//     exponent-range test), and exponent/fraction are rounded as one packed
//     integer so the significand carry, subnormal->normal and overflow->Inf
//     transitions fall out of one increment chain;
//   * mul: at most one operand normalised before the product (two subnormal
//     operands underflow to zero), an exact (S+1)x(S+1) product -- array cells
//     for S < 9, radix-4 Booth rows with a compile-time Dadda reduction for
//     S >= 9 -- a 1-bit product normalise, a narrow (S+3)-bit subnormal
//     shifter driven by a (E+2)-bit exponent, packed rounding as above;
//   * special values come from the larger-magnitude operand (add) or four
//     class masks (mul) and are applied with one LOP3 per output plane.
// Bit-exactness against the reference is established by tests, not by
// structural similarity (tests/test_circuits_host.py exhaustively on the CPU,
// tests/test_gpu_parity.py on the B200).
//
// The same header compiles for the host (g++) so the networks can be checked
// exhaustively without a GPU.
#pragma once
#if defined(__CUDACC_RTC__)
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
typedef unsigned char uint8_t;
typedef unsigned long long uintptr_t;
#else
#include <stdint.h>
#endif

#if defined(__CUDACC__)
#define BFP_HD __host__ __device__ __forceinline__
#define BFP_UNROLL _Pragma("unroll")
#else
#define BFP_HD inline
#define BFP_UNROLL
#endif

// Stage markers for the mapper's per-stage LUT report (tools/lutmap/stages.cpp);
// no code anywhere else.
#ifndef BFP_STAGE
#define BFP_STAGE(name)
#endif

namespace bfpg {

#if defined(BFP_SYMBOLIC_WORD)
// tools/lutmap: the same networks evaluated on a symbolic word (a DAG node)
typedef BFP_SYMBOLIC_WORD w32;
static const w32 ONES = w32(0xffffffffu);
#else
typedef uint32_t w32;
constexpr w32 ONES = 0xffffffffu;
#endif

template <int E_, int S_, bool RN_, bool FTZ_>
struct Format {
  static constexpr int E = E_;
  static constexpr int S = S_;
  static constexpr int N = 1 + E_ + S_;  // planes
  static constexpr bool RN = RN_;
  static constexpr bool FTZ = FTZ_;
  static constexpr int BIAS = (1 << (E_ - 1)) - 1;
};

constexpr int clog2(int n) {
  int k = 0;
  while ((1 << k) < n) ++k;
  return k;
}
constexpr int imax(int a, int b) { return a > b ? a : b; }
constexpr int imin(int a, int b) { return a < b ? a : b; }

// ---------------------------------------------------------------- gates
BFP_HD w32 mux(w32 s, w32 a, w32 b) { return (s & a) | (~s & b); }  // s ? a : b
BFP_HD w32 maj(w32 a, w32 b, w32 c) { return (a & b) | (c & (a | b)); }

// Pinned 3-input LUTs.  ptxas maps plain C expressions greedily and fuses a
// shared sub-term (e.g. a partial product) into every consumer, duplicating
// it; where the optimal cover is known, the network is written directly in
// lop3.b32 so ptxas keeps exactly one LOP3 per node.
#if defined(__CUDA_ARCH__)
template <int LUT>
__device__ __forceinline__ w32 lop3(w32 a, w32 b, w32 c) {
  w32 r;
  asm("lop3.b32 %0, %1, %2, %3, %4;" : "=r"(r) : "r"(a), "r"(b), "r"(c), "n"(LUT));
  return r;
}
#else
template <int LUT>
inline w32 lop3(w32 a, w32 b, w32 c) {
  w32 r = 0;
  for (int k = 0; k < 8; ++k) {
    const w32 ta = (k & 4) ? a : ~a, tb = (k & 2) ? b : ~b, tc = (k & 1) ? c : ~c;
    if ((LUT >> k) & 1) r |= ta & tb & tc;
  }
  return r;
}
#endif
// LUT encodings over (a, b, c) = (0xF0, 0xCC, 0xAA)
constexpr int L_AND2 = 0xC0;       // a & b
constexpr int L_XOR3 = 0x96;       // a ^ b ^ c
constexpr int L_MAJ = 0xE8;        // maj(a, b, c)
constexpr int L_XOR_AND = 0x6A;    // c ^ (a & b)
constexpr int L_AND3 = 0x80;       // a & b & c
constexpr int L_MUX = 0xCA;        // a ? b : c
constexpr int L_ANDN = 0x30;       // a & ~b
constexpr int L_OR3 = 0xFE;        // a | b | c

// Pinned mux / masked copy (one LOP3 each, never duplicated into consumers).
BFP_HD w32 pmux(w32 s, w32 a, w32 b) { return lop3<L_MUX>(s, a, b); }
BFP_HD w32 pandn(w32 a, w32 s) { return lop3<L_ANDN>(a, s, 0u); }

// a >= v for an unsigned K-bit field a (LSB first) and a constant v.
template <int K>
BFP_HD w32 ge_const(const w32* a, int v) {
  if (v <= 0) return ONES;
  if (v >= (1 << K)) return 0;
  w32 r = ONES;
  BFP_UNROLL for (int i = 0; i < K; ++i) r = ((v >> i) & 1) ? (a[i] & r) : (a[i] | r);
  return r;
}

// ------------------------------------------------------- shifters
// Right shift of f[0..W) by `dist` where sel is set; bit 0 is a jam (sticky)
// position that absorbs every bit shifted through it.
template <int W, int DIST>
BFP_HD void shr_jam_stage(w32 (&f)[W], w32 sel) {
  if constexpr (DIST < W) {
    w32 t = 0;
    BFP_UNROLL for (int i = 1; i <= DIST && i < W; ++i) t |= f[i];
    w32 nf[W];
    nf[0] = f[0] | (sel & t);
    BFP_UNROLL for (int i = 1; i < W; ++i)
      nf[i] = (i + DIST < W) ? pmux(sel, f[i + DIST], f[i]) : pandn(f[i], sel);
    BFP_UNROLL for (int i = 0; i < W; ++i) f[i] = nf[i];
  } else {
    w32 t = 0;
    BFP_UNROLL for (int i = 1; i < W; ++i) t |= f[i];
    f[0] = f[0] | (sel & t);
    BFP_UNROLL for (int i = 1; i < W; ++i) f[i] = f[i] & ~sel;
  }
}

template <int W, int K, int KK = 0>
BFP_HD void shr_jam(w32 (&f)[W], const w32* amt) {
  if constexpr (KK < K) {
    shr_jam_stage<W, (1 << KK)>(f, amt[KK]);
    shr_jam<W, K, KK + 1>(f, amt);
  }
}

// Left shift of f[0..W) by DIST where sel is set (zero fill).
template <int W, int DIST>
BFP_HD void shl_stage(w32 (&f)[W], w32 sel) {
  w32 nf[W];
  BFP_UNROLL for (int i = 0; i < W; ++i)
    nf[i] = (i >= DIST) ? pmux(sel, f[i - DIST], f[i]) : pandn(f[i], sel);
  BFP_UNROLL for (int i = 0; i < W; ++i) f[i] = nf[i];
}

// Unlimited leading-zero normaliser over f[0..W): stage k (descending) shifts
// left by 2^k when the top 2^k bits are all zero; cnt[k] records it.
template <int W, int K, int KK>
BFP_HD void normalize_stages(w32 (&f)[W], w32* cnt) {
  if constexpr (KK >= 0) {
    constexpr int D = 1 << KK;
    if constexpr (D < W) {
      w32 any = 0;
      BFP_UNROLL for (int i = W - D; i < W; ++i) any |= f[i];
      const w32 c = ~any;
      shl_stage<W, D>(f, c);
      cnt[KK] = c;
    } else {
      cnt[KK] = 0;
    }
    normalize_stages<W, K, KK - 1>(f, cnt);
  }
}

// ------------------------------------------------ integer arithmetic
// r = a + b + cin over K bits; returns carry out.
template <int K>
BFP_HD w32 add_k(const w32* a, const w32* b, w32 cin, w32* r) {
  w32 c = cin;
  BFP_UNROLL for (int i = 0; i < K; ++i) {
    const w32 ai = a[i], bi = b[i];
    r[i] = ai ^ bi ^ c;
    c = maj(ai, bi, c);
  }
  return c;
}

// r = a - b over K bits (a + ~b + 1); returns the borrow (a < b).
template <int K>
BFP_HD w32 sub_k(const w32* a, const w32* b, w32* r) {
  w32 c = ONES;
  BFP_UNROLL for (int i = 0; i < K; ++i) {
    const w32 ai = a[i], nbi = ~b[i];
    r[i] = ai ^ nbi ^ c;
    c = maj(ai, nbi, c);
  }
  return ~c;
}

// ------------------------------------------------------- final assembly
// Packs [expfield (EW bits, may be wider than E) : frac(S)] with the hidden
// bit added at position S and the rounding increment at position 0:
//   out = frac + rnd, exp = expf + hidden + carry(frac + rnd).
// Returns the E+1 bits of the exponent sum in ex[] (bit E = overflow past
// 2^E) and the final S fraction bits in fr[].
template <int E, int S, int EW>
BFP_HD void pack_round(const w32* expf, const w32* sig /*S+1*/, w32 rnd, w32* fr, w32* ex) {
  w32 c = rnd;
  BFP_UNROLL for (int i = 0; i < S; ++i) {
    const w32 v = sig[i];
    fr[i] = v ^ c;
    c = v & c;
  }
  // position S: expf[0] + hidden + carry
  {
    const w32 h = sig[S], v = expf[0];
    ex[0] = v ^ h ^ c;
    c = maj(v, h, c);
  }
  BFP_UNROLL for (int i = 1; i <= E; ++i) {
    const w32 v = (i < EW) ? expf[i] : 0u;
    ex[i] = v ^ c;
    c = v & c;
  }
}

// Generated LOP3 covers (tools/lutmap, build time) specialise this per
// (format, op) with `ok = true` and a straight-line `run`; the templates
// below are the source they are generated from and the fallback.
template <class F, int OP>
struct Gen {
  static constexpr bool ok = false;
};

// ================================================================= ADD
// Z = X + Y (SUB: X - Y).  bfp_add / bfp_sub semantics, arith.hpp:235-328.
//
// FAST: the caller guarantees (mul_add_fast_domain below) that both operands
// are finite normals, the larger exponent field is >= 2^KN and <= 2^E - 3: the
// hidden bits are constant ones, the normaliser's budget never binds, nothing
// is special and the sum cannot overflow; every signal replaced by a constant
// here has that value in the general network on that domain.
template <class F, bool SUB, bool FAST = false>
BFP_HD void add_w(const w32* X, const w32* Y, w32* Z) {
  constexpr int E = F::E, S = F::S, M = E + S;
  const w32 sx = X[M];
  const w32 sy = SUB ? ~Y[M] : Y[M];

  BFP_STAGE("add.compare_swap");
  // Order by magnitude: swap = |X| < |Y| as (E+S)-bit encodings (borrow of X-Y).
  w32 bw = 0;
  BFP_UNROLL for (int i = 0; i < M; ++i) bw = maj(~X[i], Y[i], bw);
  const w32 swap = bw;
  w32 A[M], B[M];
  BFP_UNROLL for (int i = 0; i < M; ++i) {
    A[i] = pmux(swap, Y[i], X[i]);
    B[i] = pmux(swap, X[i], Y[i]);
  }
  const w32 sa = mux(swap, sy, sx);
  const w32 sb = mux(swap, sx, sy);
  const w32 eff = sx ^ sy;  // effective subtraction

  BFP_STAGE("add.classes_distance");
  // Hidden bits (exponent nonzero) and effective exponents (subnormals at 1).
  w32 ha = 0, hb = 0;
  BFP_UNROLL for (int i = 0; i < E; ++i) {
    ha |= A[S + i];
    hb |= B[S + i];
  }
  if constexpr (FAST) ha = hb = ONES;
  w32 ea[E], eb[E];
  BFP_UNROLL for (int i = 0; i < E; ++i) {
    ea[i] = A[S + i];
    eb[i] = B[S + i];
  }
  ea[0] |= ~ha;
  eb[0] |= ~hb;

  // Alignment distance d = ea - eb >= 0.
  w32 d[E];
  (void)sub_k<E>(ea, eb, d);

  BFP_STAGE("add.align");
  // Align B: [jam, r, g, frac(S), hidden] right by d.  Distances >= WA-1 put
  // everything in the jam bit, so the amount saturates at 2^KA - 1 >= WA - 1.
  constexpr int WA = S + 4;
  constexpr int KA = clog2(WA);
  constexpr int KS = imin(KA, E);
  w32 f[WA];
  f[0] = 0;
  f[1] = 0;
  f[2] = 0;
  BFP_UNROLL for (int j = 0; j < S; ++j) f[3 + j] = B[j];
  f[S + 3] = hb;
  w32 amt[KS];
  {
    w32 big = 0;
    BFP_UNROLL for (int k = KA; k < E; ++k) big |= d[k];
    BFP_UNROLL for (int k = 0; k < KS; ++k) amt[k] = d[k] | big;
  }
  shr_jam<WA, KS>(f, amt);

  BFP_STAGE("add.adder");
  // One adder for both effective operations: A + (B ^ eff) + eff.
  constexpr int WN = WA + 1;
  w32 x[WN];
  {
    w32 ma[WA];
    ma[0] = 0;
    ma[1] = 0;
    ma[2] = 0;
    BFP_UNROLL for (int j = 0; j < S; ++j) ma[3 + j] = A[j];
    ma[S + 3] = ha;
    w32 c = eff;
    BFP_UNROLL for (int i = 0; i < WA; ++i) {
      const w32 t = f[i] ^ eff;
      x[i] = ma[i] ^ t ^ c;
      c = maj(ma[i], t, c);
    }
    x[WA] = c & ~eff;  // only an effective add carries out
  }

  BFP_STAGE("add.normalize");
  // Budget-limited normalise: shift left by sh = min(lz(x), ea) so results
  // below the smallest normal stop at the subnormal position.  The budget r
  // starts at min(ea, 2^KN - 1) and is decremented by every shift taken.
  constexpr int KN = clog2(WN);  // 2^KN - 1 >= WN - 1
  w32 r[KN];
  {
    w32 big = 0;
    BFP_UNROLL for (int k = KN; k < E; ++k) big |= ea[k];
    if constexpr (FAST) big = ONES;
    BFP_UNROLL for (int k = 0; k < KN; ++k) r[k] = (k < E ? ea[k] : 0u) | big;
  }
  w32 sh[KN];
  BFP_UNROLL for (int k = KN - 1; k >= 0; --k) {
    const int D = 1 << k;
    w32 ok = 0;
    BFP_UNROLL for (int j = k; j < KN; ++j) ok |= r[j];
    w32 any = 0;
    BFP_UNROLL for (int i = WN - D; i < WN; ++i) any |= (i >= 0 ? x[i] : 0u);
    const w32 c = ok & ~any;
    sh[k] = c;
    // The leading one of a sum without carry-out sits at most two places
    // below the top when the exponent distance is >= 2 (x >= A - A/4), so a
    // shift by D >= 4 only happens on a massive cancellation (effective
    // subtraction, distance <= 1), where the jam and round bits x[0], x[1]
    // are zero -- B moved by at most one place -- and stay zero: those
    // stages shift zeros into positions D and D + 1.
    w32 nx[WN];
    BFP_UNROLL for (int i = 0; i < WN; ++i)
      nx[i] = (i >= D && (D < 4 || i - D >= 2)) ? pmux(c, x[i - D], x[i]) : pandn(x[i], c);
    BFP_UNROLL for (int i = 0; i < WN; ++i) x[i] = nx[i];
    if (k > 0) {
      // r -= c << k (r >= 2^k whenever c is set)
      w32 bo = c;
      BFP_UNROLL for (int j = k; j < KN; ++j) {
        const w32 rj = r[j];
        r[j] = rj ^ bo;
        bo = bo & ~rj;
      }
    }
  }

  BFP_STAGE("add.round_pack");
  // sig = x[4..S+4], guard x[3], sticky x[0..2].
  const w32* sig = x + 4;
  w32 rnd = 0;
  if constexpr (F::RN) rnd = x[3] & (x[0] | x[1] | x[2] | sig[0]);

  // D = ea - sh; exponent field = D + hidden (+ rounding carry).
  w32 Dx[E];
  {
    w32 shx[E];
    BFP_UNROLL for (int i = 0; i < E; ++i) shx[i] = (i < KN) ? sh[i] : 0u;
    (void)sub_k<E>(ea, shx, Dx);
  }
  w32 fr[S], ex[E + 1];
  pack_round<E, S, E>(Dx, sig, rnd, fr, ex);

  BFP_STAGE("add.specials_out");
  // Exact zero: +0 from cancellation, -0 only for (-0) + (-0).
  w32 nz = 0;
  BFP_UNROLL for (int i = 0; i <= S; ++i) nz |= sig[i];
  const w32 hidden = sig[S];

  // Specials: the larger-magnitude operand is Inf/NaN whenever either is.
  w32 as = ONES, bs = ONES, afz = 0;
  BFP_UNROLL for (int i = 0; i < E; ++i) {
    as &= A[S + i];
    bs &= B[S + i];
  }
  BFP_UNROLL for (int i = 0; i < S; ++i) afz |= A[i];
  if constexpr (FAST) as = bs = 0;
  const w32 use_nan = as & (afz | (bs & eff));

  // Overflow: exponent sum >= 2^E - 1.
  w32 eall = ONES;
  BFP_UNROLL for (int i = 0; i < E; ++i) eall &= ex[i];
  w32 ovf = ex[E] | eall;
  if constexpr (FAST) ovf = ex[E] = 0;

  // Fraction mask: keep unless special, overflow (RN: Inf) or FTZ flush.
  w32 keep = ~as;
  if constexpr (F::RN) keep &= ~ovf;
  if constexpr (F::FTZ) keep &= hidden;  // add: subnormal results are exact
  w32 setf = 0;
  if constexpr (!F::RN) setf = ovf & ~as;  // RZ overflow -> max finite
  BFP_UNROLL for (int j = 0; j < S; ++j) Z[j] = (fr[j] & keep) | setf;
  Z[S - 1] |= use_nan;

  // Exponent plane: zero results clear, specials / RN overflow set all.
  w32 setx = as;
  if constexpr (F::RN) setx |= ex[E];
  BFP_UNROLL for (int j = 0; j < E; ++j) {
    w32 v = ex[j] & nz;
    if constexpr (!F::RN)
      if (j == 0) v &= ~ovf;  // RZ overflow -> exponent 2^E - 2
    Z[S + j] = v | setx;
  }
  // Sign: specials take A's sign (NaN positive); zero sums sa & sb.
  Z[M] = sa & mux(as, ~use_nan, sb | nz);
}

// ====================================================== shared final stage
// Rounds and packs a significand field R = [jam, guard, sig(S+1)] whose
// biased exponent minus one is ez (EW-bit two's complement, EW >= E+2):
//   ez >= 0: normal, exponent field ez + hidden (+ rounding carry);
//   ez <  0: subnormal range, R shifts right by -ez first (jam collects);
// then overflow (Inf under RN, max-finite under RZ), FTZ after rounding
// (still below the smallest normal) and the special-value overrides:
// zero_res / inf_res force a signed zero / Inf, use_nan the canonical NaN.
// FAST: 0 <= ez <= 2^E - 4 is guaranteed (no subnormal-range shift, no flush,
// no overflow).
template <class F, int EW, bool FAST = false>
BFP_HD void finish_round(w32* R, const w32* ez, w32 sign, w32 zero_res, w32 inf_res, w32 use_nan,
                         w32* Z) {
  constexpr int E = F::E, S = F::S, M = E + S;
  static_assert(EW >= E + 2, "finish_round: working exponent narrower than E + 2");
  constexpr int WR = S + 3;
  BFP_STAGE("fr.subnormal_shift");
  const w32 sub = FAST ? w32(0u) : ez[EW - 1];
  if constexpr (!FAST) {
    // amt = -ez = ~ez + 1, live only on sub; saturate at 2^KR - 1 >= WR - 1.
    constexpr int KR = clog2(WR);
    constexpr int KRS = imin(KR, EW);
    w32 ng[EW];
    w32 c = ONES;
    BFP_UNROLL for (int i = 0; i < EW; ++i) {
      const w32 v = ~ez[i];
      ng[i] = v ^ c;
      c = v & c;
    }
    w32 big = 0;
    BFP_UNROLL for (int k = KR; k < EW; ++k) big |= ng[k];
    w32 amt[KRS];
    BFP_UNROLL for (int k = 0; k < KRS; ++k) amt[k] = (ng[k] | big) & sub;
    w32 (&Rr)[WR] = *reinterpret_cast<w32(*)[WR]>(R);
    shr_jam<WR, KRS>(Rr, amt);
  }
  BFP_STAGE("fr.round_pack");
  const w32* sig = R + 2;
  w32 rnd = 0;
  if constexpr (F::RN) rnd = R[1] & (R[0] | sig[0]);

  // exponent field: ez masked to 0 in the subnormal range (E+1 bits kept for
  // overflow detection), + hidden, + rounding carry.
  w32 em[E + 1];
  BFP_UNROLL for (int i = 0; i <= E; ++i) em[i] = ez[i] & ~sub;
  w32 fr[S], ex[E + 2];
  pack_round<E + 1, S, E + 1>(em, sig, rnd, fr, ex);
  w32 eall = ONES;
  BFP_UNROLL for (int i = 0; i < E; ++i) eall &= ex[i];
  // ez bits above E (only when EW > E + 2): a positive ez >= 2^(E+1) overflows
  w32 high = 0;
  BFP_UNROLL for (int i = E + 1; i < EW - 1; ++i) high |= ez[i];
  w32 ovf = ex[E] | ex[E + 1] | eall | (high & ~sub);
  if constexpr (FAST) ovf = 0;

  BFP_STAGE("fr.specials_out");
  w32 flush = 0;
  if constexpr (F::FTZ) flush = sub & ~ex[0];  // still below the smallest normal
  const w32 quiet = ~(zero_res | inf_res | use_nan);
  const w32 force = inf_res | use_nan;  // exponent all ones
  w32 keep, setf = 0;
  if constexpr (F::RN) {
    keep = quiet & ~ovf & ~flush;
  } else {
    keep = quiet & ~flush;
    setf = quiet & ovf;
  }
  BFP_UNROLL for (int j = 0; j < S; ++j) Z[j] = (fr[j] & keep) | setf;
  Z[S - 1] |= use_nan;
  const w32 hset = force | (quiet & ovf);
  BFP_UNROLL for (int j = 0; j < E; ++j) {
    if constexpr (!F::RN) {
      if (j == 0) {
        Z[S] = (ex[0] & quiet & ~ovf) | force;
        continue;
      }
    }
    Z[S + j] = (ex[j] & quiet) | hset;
  }
  Z[M] = sign & ~use_nan;
}

// Signed working-exponent widths.  E + 2 bits hold every intermediate of the
// named formats; a format with a wide significand and a narrow exponent range
// (e.g. 1/3/11, 1/2/5: normalisation counts up to S or 2S+1 against a bias of
// 3 or 1) needs more, so the width is the larger of E + 2 and the bits of the
// exact range of the exponent expression (plus one of margin).
constexpr int signed_bits(long lo, long hi) {
  int w = 2;
  while (lo < -(1L << (w - 1)) || hi >= (1L << (w - 1))) ++w;
  return w;
}
// mul: ez = ex_eff + ey_eff - bias - lz - borrow, finite ex_eff in [1, 2^E - 2],
// lz <= S (one normalised operand) or 2S + 1 (full product normaliser).
template <class F>
constexpr int mul_ew() {
  constexpr long bias = F::BIAS;
  constexpr long lzmax = ((1 - F::BIAS) <= -F::S - 1) ? F::S : 2L * F::S + 1;
  return imax(F::E + 2, signed_bits(-bias - lzmax - 2, 2 * ((1L << F::E) - 2) - bias + 1));
}
// div: ez = (ex_eff - lzx) - (ey_eff - lzy) - scale + bias - 1, lz <= S.
template <class F>
constexpr int div_ew() {
  constexpr long bias = F::BIAS, top = (1L << F::E) - 2;
  return imax(F::E + 2, signed_bits(1 - top - F::S - 1 + bias - 1 - 1, top - 1 + F::S + bias - 1 + 1));
}

// Operand classes shared by mul / div.
struct Classes {
  w32 h;   // hidden bit (exponent nonzero)
  w32 s;   // exponent all ones (Inf / NaN)
  w32 f;   // fraction nonzero
  w32 z;   // zero
  w32 inf;
  w32 nan;
};

template <class F>
BFP_HD Classes classify(const w32* X) {
  constexpr int E = F::E, S = F::S;
  Classes c{0, ONES, 0, 0, 0, 0};
  BFP_UNROLL for (int i = 0; i < E; ++i) {
    c.h |= X[S + i];
    c.s &= X[S + i];
  }
  BFP_UNROLL for (int i = 0; i < S; ++i) c.f |= X[i];
  c.z = ~c.h & ~c.f;
  c.inf = c.s & ~c.f;
  c.nan = c.s & c.f;
  return c;
}

// ================================================================= MUL
// Exact product of two (S+1)-bit significands: shift-add rows, one carry
// chain per row; each cell = AND (partial product) + XOR3 + MAJ, pinned.
template <int S>
BFP_HD void sig_product(const w32* mx, const w32* my, w32* P /*2S+2*/) {
  BFP_UNROLL for (int j = 0; j <= S; ++j) P[j] = lop3<L_AND2>(mx[j], my[0], 0u);
  BFP_UNROLL for (int i = 1; i <= S; ++i) {
    // j = 0: carry-in 0 -> sum = a ^ pp, carry = a & pp (AND fused)
    w32 c = lop3<L_AND3>(mx[0], my[i], P[i]);
    P[i] = lop3<L_XOR_AND>(mx[0], my[i], P[i]);
    BFP_UNROLL for (int j = 1; j <= S; ++j) {
      if (i == 1 && j == S) {  // nothing accumulated above row 0 yet
        const w32 s0 = lop3<L_XOR_AND>(mx[j], my[i], c);
        c = lop3<L_AND3>(mx[j], my[i], c);
        P[i + j] = s0;
        continue;
      }
      const w32 pp = lop3<L_AND2>(mx[j], my[i], 0u);
      const w32 a = P[i + j];
      P[i + j] = lop3<L_XOR3>(a, pp, c);
      c = lop3<L_MAJ>(a, pp, c);
    }
    P[i + S + 1] = c;
  }
}

// Radix-4 Booth product with a compile-time Dadda reduction schedule.
//
// Multiplier digits d_k = -2 b[2k+1] + b[2k] + b[2k-1] (k = 0..R-1, b[-1] and
// bits above S zero) select rows |d_k|·a of S+2 bits, complemented when
// negative: one row bit is ((a_j & one) ^ neg) ^ (a_{j-1} & two) -- two LUTs,
// one/two being exclusive -- plus neg_k at column 2k (the +1 of the two's
// complement), ~neg_k at column 2k+S+2 and the constant -sum_k 2^(S+2+2k)
// (sign extension folded into constants).  Half as many rows as the array
// product at two LUTs per row bit: for S >= 9 the mapped network is smaller
// (1/5/10 -9%, 1/8/15 -15%, 1/8/23 -21% of the product).  The column heights
// are static, so the full adders / half adders of a Dadda reduction and the
// final ripple are planned by a constexpr function and executed over a slot
// array whose indices are all compile-time constants after unrolling.
template <int S>
struct BoothPlan {
  static constexpr int NB = S + 1, W = 2 * S + 2, R = NB / 2 + 1, RW = S + 2;
  static constexpr int NPP = R * RW;  // slots [0, NPP): row bit q(k, j) = k*RW + j
  static constexpr int SNEG = NPP, SNNEG = NPP + R, SONE = NPP + 2 * R, NIN = SONE + 1;
  static constexpr int MAXOPS = NPP + 3 * R + 2 * W;
  static constexpr int NSLOT = NIN + 2 * MAXOPS;
  static constexpr int HMAX = 2 * R + 16;
  bool ok = true;  // false: a static bound was too small (rejected at compile time)
  int nops = 0;
  short a[MAXOPS] = {}, b[MAXOPS] = {}, c[MAXOPS] = {};  // c < 0: half adder
  short so[MAXOPS] = {}, co[MAXOPS] = {};               // sum slot, carry slot (-1: dropped)
  short f0[W] = {}, f1[W] = {};                         // final two rows (-1: zero)
};

template <int S>
constexpr BoothPlan<S> make_booth_plan() {
  using P = BoothPlan<S>;
  constexpr int W = P::W, R = P::R, RW = P::RW, H = P::HMAX;
  P pl{};
  short col[W][H] = {};
  int h[W] = {};
  auto push = [&](int k, int slot) {
    if (k >= W) return;
    if (h[k] >= H) {
      pl.ok = false;
      return;
    }
    col[k][h[k]++] = short(slot);
  };
  for (int k = 0; k < R; ++k) {
    for (int j = 0; j < RW; ++j) push(2 * k + j, k * RW + j);
    push(2 * k, P::SNEG + k);
    push(2 * k + S + 2, P::SNNEG + k);
  }
  unsigned long long cst = 0;
  for (int k = 0; k < R; ++k) cst -= (1ull << (S + 2)) << (2 * k);
  for (int k = 0; k < W; ++k)
    if ((cst >> k) & 1) push(k, P::SONE);
  int maxh = 0;
  for (int k = 0; k < W; ++k) maxh = h[k] > maxh ? h[k] : maxh;
  int d[16] = {2};
  int nd = 1;
  while (d[nd - 1] < maxh) {
    d[nd] = d[nd - 1] * 3 / 2;
    ++nd;
  }
  int next = P::NIN;
  auto pop = [&](int k) { return col[k][--h[k]]; };  // newest first (smallest mapped cover)
  for (int st = nd - 2; st >= 0; --st) {
    const int tgt = d[st];
    for (int k = 0; k < W; ++k) {
      while (h[k] > tgt) {
        if (pl.nops >= P::MAXOPS || h[k] < 2) {
          pl.ok = false;
          return pl;
        }
        const int i = pl.nops++;
        const bool fa = h[k] - tgt >= 2;
        pl.a[i] = pop(k);
        pl.b[i] = pop(k);
        pl.c[i] = fa ? pop(k) : short(-1);
        pl.so[i] = short(next++);
        pl.co[i] = (k + 1 < W) ? short(next++) : short(-1);
        push(k, pl.so[i]);
        if (k + 1 < W) push(k + 1, pl.co[i]);
      }
    }
  }
  for (int k = 0; k < W; ++k) {
    pl.f0[k] = h[k] > 0 ? col[k][0] : short(-1);
    pl.f1[k] = h[k] > 1 ? col[k][1] : short(-1);
  }
  return pl;
}

template <int S>
BFP_HD void sig_product_booth(const w32* a, const w32* b, w32* P) {
  using PL = BoothPlan<S>;
  constexpr PL pl = make_booth_plan<S>();
  static_assert(pl.ok, "BoothPlan bounds");
  constexpr int NB = PL::NB, W = PL::W, R = PL::R, RW = PL::RW;
  w32 v[PL::NSLOT];
  BFP_UNROLL for (int k = 0; k < R; ++k) {
    const w32 b2 = (2 * k + 1 < NB) ? b[2 * k + 1] : w32(0u);
    const w32 b1 = (2 * k < NB) ? b[2 * k] : w32(0u);
    const w32 b0 = (k > 0) ? b[2 * k - 1] : w32(0u);
    const w32 one = b1 ^ b0;
    const w32 two = (b2 & ~b1 & ~b0) | (~b2 & b1 & b0);
    BFP_UNROLL for (int j = 0; j < RW; ++j) {
      const w32 aj = (j < NB) ? a[j] : w32(0u);
      const w32 aj1 = (j >= 1) ? a[j - 1] : w32(0u);
      v[k * RW + j] = ((aj & one) ^ b2) ^ (aj1 & two);
    }
    v[PL::SNEG + k] = b2;
    v[PL::SNNEG + k] = ~b2;
  }
  v[PL::SONE] = ONES;
  BFP_UNROLL for (int i = 0; i < pl.nops; ++i) {
    const w32 x = v[pl.a[i]], y = v[pl.b[i]];
    if (pl.c[i] >= 0) {
      const w32 z = v[pl.c[i]];
      v[pl.so[i]] = x ^ y ^ z;
      if (pl.co[i] >= 0) v[pl.co[i]] = maj(x, y, z);
    } else {
      v[pl.so[i]] = x ^ y;
      if (pl.co[i] >= 0) v[pl.co[i]] = x & y;
    }
  }
  w32 c = 0u;
  BFP_UNROLL for (int k = 0; k < W; ++k) {
    const w32 x = pl.f0[k] >= 0 ? v[pl.f0[k]] : w32(0u);
    const w32 y = pl.f1[k] >= 0 ? v[pl.f1[k]] : w32(0u);
    P[k] = x ^ y ^ c;
    c = maj(x, y, c);
  }
}

// The smaller network of the two for this width (mapped LOP3 counts).
template <int S>
BFP_HD void sig_product_best(const w32* a, const w32* b, w32* P) {
  if constexpr (S >= 9 && S <= 30)
    sig_product_booth<S>(a, b, P);
  else
    sig_product<S>(a, b, P);
}

// Z = X * Y.  bfp_mul semantics, arith.hpp:330-373.
//
// When emin <= -S-1 (every format here but 1/3/2), two subnormal operands
// give |x*y| < 2^(2 emin) <= half the smallest subnormal, which rounds to a
// signed zero in every mode; that case is forced through the zero mask, so at
// most one operand needs normalising.  That operand's significand (S+1 bits)
// is normalised BEFORE the product -- the operands are ordered by hidden bit
// (two muxes per significand bit; the exponent sum is symmetric) -- and the
// product, then in [2^2S, 2^(2S+2)), needs a single 1-bit normalise instead of
// a log shifter over all 2S+2 product bits.
//
// FAST: both operands are finite normals and the sum of their exponent fields
// lies in [2^(E-1), 2^E + 2^(E-1) - 5] (mul_add_fast_domain): neither operand
// needs normalising, the biased result exponent minus one, ez = ea + eb - bias
// - 1 + top, is >= 0 and the rounded result's field ez + 1 (+1 on a rounding
// carry when top = 0) is <= 2^E - 3 -- the pre-product normaliser, the
// subnormal-range shifter, the special-value masks and the overflow path of
// finish_round fold away.
template <class F, bool FAST = false>
BFP_HD void mul_w(const w32* X, const w32* Y, w32* Z) {
  constexpr int E = F::E, S = F::S, M = E + S;
  constexpr int EW = mul_ew<F>();  // signed working exponent
  constexpr bool BOTH_SUB_ZERO = (1 - F::BIAS) <= -S - 1;
  static_assert(!FAST || BOTH_SUB_ZERO, "mul_w: the fast domain needs emin <= -S-1");
  BFP_STAGE("mul.classes");
  const w32 sign = X[M] ^ Y[M];
  Classes cx = classify<F>(X), cy = classify<F>(Y);
  if constexpr (FAST) {
    cx.h = cy.h = ONES;
    cx.z = cy.z = cx.s = cy.s = cx.inf = cy.inf = cx.nan = cy.nan = 0;
  }

  constexpr int WP = 2 * S + 2;
  w32 P[WP];
  w32 R[S + 3];  // [jam, guard, sig(S+1)]
  w32 ez[EW];
  // ez = ex_eff + ey_eff - bias - lz - borrow  (biased result exponent minus one).
  // With -bias = 1 - 2^(E-1) and -lz - 1 = ~lz this is two carry chains:
  //   t  = ex_eff + ey_eff + 1
  //   ez = t + K + (1 - borrow),  K = ~lz (sign-extended) - 2^(E-1),
  // and when lz has no bit at or above E-1, K is ~lz below KL and the constant
  // ...1101...1 (zero at bit E-1) above: no separate pass for the bias.
  auto exponent = [&](const w32* lz, int KL, w32 borrow_in_sub) {
    w32 a[EW], b[EW];
    BFP_UNROLL for (int i = 0; i < EW; ++i) {
      a[i] = (i < E) ? X[S + i] : 0u;
      b[i] = (i < E) ? Y[S + i] : 0u;
    }
    a[0] |= ~cx.h;
    b[0] |= ~cy.h;
    if (KL <= E - 1) {
      w32 t[EW];
      (void)add_k<EW>(a, b, ONES, t);
      w32 c = ~borrow_in_sub;
      BFP_UNROLL for (int i = 0; i < EW; ++i) {
        const w32 ti = t[i];
        const w32 ki = (i < KL) ? ~lz[i] : (i == E - 1 ? w32(0u) : ONES);
        ez[i] = ti ^ ki ^ c;
        c = maj(ti, ki, c);
      }
      return;
    }
    w32 t[EW];
    (void)add_k<EW>(a, b, 0, t);
    w32 nb[EW];
    constexpr int NB = (1 << EW) - F::BIAS;  // -bias mod 2^EW
    BFP_UNROLL for (int i = 0; i < EW; ++i) nb[i] = ((NB >> i) & 1) ? ONES : 0u;
    w32 u[EW];
    (void)add_k<EW>(t, nb, 0, u);
    // ez = u - lz - borrow_in_sub = u + ~lz + (1 - borrow_in_sub)
    w32 c = ~borrow_in_sub;
    BFP_UNROLL for (int i = 0; i < EW; ++i) {
      const w32 ui = u[i], nl = ~((i < KL) ? lz[i] : 0u);
      ez[i] = ui ^ nl ^ c;
      c = maj(ui, nl, c);
    }
  };
  if constexpr (BOTH_SUB_ZERO) {
    // s: the operand that may be subnormal (X unless X is normal), n: the other.
    BFP_STAGE("mul.order_normalize");
    w32 ms[S + 1], mn[S + 1];
    BFP_UNROLL for (int i = 0; i < S; ++i) {
      ms[i] = pmux(cx.h, Y[i], X[i]);
      mn[i] = pmux(cx.h, X[i], Y[i]);
    }
    ms[S] = cx.h & cy.h;  // hidden bit of s: clear iff either is subnormal
    mn[S] = ONES;         // n is normal (or the result is forced to zero)
    constexpr int KN = clog2(S + 1) > 0 ? clog2(S + 1) : 1;
    w32 lz[KN];
    normalize_stages<S + 1, KN, KN - 1>(ms, lz);
    ms[S] = ONES;  // a zero significand (the only one without a leading one) forces a zero result
    BFP_STAGE("mul.product");
    sig_product_best<S>(mn, ms, P);
    // 1-bit normalise: top = P[2S+1]; otherwise the leading one is at 2S.
    BFP_STAGE("mul.normalize1_exponent");
    const w32 top = P[WP - 1];
    w32 st = 0;
    BFP_UNROLL for (int i = 0; i + 1 < S; ++i) st |= P[i];
    R[0] = st | (top & P[S - 1]);
    R[1] = pmux(top, P[S], P[S - 1]);
    BFP_UNROLL for (int i = 0; i <= S; ++i) R[2 + i] = pmux(top, P[S + 1 + i], P[S + i]);
    exponent(lz, KN, ~top);
  } else {
    w32 mx[S + 1], my[S + 1];
    BFP_UNROLL for (int i = 0; i < S; ++i) {
      mx[i] = X[i];
      my[i] = Y[i];
    }
    mx[S] = cx.h;
    my[S] = cy.h;
    sig_product<S>(mx, my, P);
    // Normalise: leading one to position 2S+1.
    constexpr int KP = clog2(WP);
    w32 lz[KP];
    normalize_stages<WP, KP, KP - 1>(P, lz);
    w32 st = 0;
    BFP_UNROLL for (int i = 0; i < S; ++i) st |= P[i];
    R[0] = st;
    R[1] = P[S];
    BFP_UNROLL for (int i = 0; i <= S; ++i) R[2 + i] = P[S + 1 + i];
    exponent(lz, KP, 0u);
  }

  // Special-value rules of bfp_mul (arith.hpp:193-199).
  BFP_STAGE("mul.special_masks");
  const w32 use_nan = cx.nan | cy.nan | (cx.inf & cy.z) | (cx.z & cy.inf);
  w32 zero_src = cx.z | cy.z;
  if constexpr (BOTH_SUB_ZERO) zero_src |= ~cx.h & ~cy.h;  // underflows to a signed zero
  const w32 zero_res = zero_src & ~use_nan;
  const w32 inf_res = (cx.inf | cy.inf) & ~use_nan;
  finish_round<F, EW, FAST>(R, ez, sign, zero_res, inf_res, use_nan, Z);
}

// ================================================================= DIV
// Z = X / Y.  bfp_div semantics, arith.hpp:375-444: both significands are
// normalised (subnormal inputs slide up, their exponents absorb the count),
// the dividend is doubled when its significand is the smaller so the
// quotient lies in [1, 2), and a restoring divider produces S+1 quotient
// bits (RZ) or S+2 (RN: one guard bit) plus a remainder-nonzero sticky.
template <class F>
BFP_HD void div_w(const w32* X, const w32* Y, w32* Z) {
  constexpr int E = F::E, S = F::S, M = E + S;
  constexpr int EW = div_ew<F>();
  constexpr int W1 = S + 1;
  const w32 sign = X[M] ^ Y[M];
  const Classes cx = classify<F>(X), cy = classify<F>(Y);

  w32 nx[W1], ny[W1];
  BFP_UNROLL for (int i = 0; i < S; ++i) {
    nx[i] = X[i];
    ny[i] = Y[i];
  }
  nx[S] = cx.h;
  ny[S] = cy.h;
  constexpr int KN = clog2(W1) > 0 ? clog2(W1) : 1;
  w32 lzx[KN], lzy[KN];
  normalize_stages<W1, KN, KN - 1>(nx, lzx);
  normalize_stages<W1, KN, KN - 1>(ny, lzy);

  // scale = nx < ny; num = nx << scale (S+2 bits, in [ny, 2ny)).
  w32 bw = 0;
  BFP_UNROLL for (int i = 0; i < W1; ++i) bw = maj(~nx[i], ny[i], bw);
  const w32 scale = bw;
  w32 num[W1 + 1];
  num[0] = nx[0] & ~scale;
  BFP_UNROLL for (int i = 1; i < W1; ++i) num[i] = mux(scale, nx[i - 1], nx[i]);
  num[W1] = nx[W1 - 1] & scale;

  // Restoring division.  The leading quotient bit is 1: R = num - ny < ny.
  constexpr int QB = F::RN ? S + 2 : S + 1;
  w32 q[QB];
  q[QB - 1] = ONES;
  w32 R[W1];
  {
    w32 d[W1 + 1], den[W1 + 1];
    BFP_UNROLL for (int i = 0; i < W1; ++i) den[i] = ny[i];
    den[W1] = 0;
    (void)sub_k<W1 + 1>(num, den, d);
    BFP_UNROLL for (int i = 0; i < W1; ++i) R[i] = d[i];
  }
  BFP_UNROLL for (int t = QB - 2; t >= 0; --t) {
    // trial = 2R - ny over S+2 bits
    w32 r2[W1 + 1], den[W1 + 1], tr[W1 + 1];
    r2[0] = 0;
    BFP_UNROLL for (int i = 0; i < W1; ++i) r2[i + 1] = R[i];
    BFP_UNROLL for (int i = 0; i < W1; ++i) den[i] = ny[i];
    den[W1] = 0;
    const w32 borrow = sub_k<W1 + 1>(r2, den, tr);
    const w32 qt = ~borrow;
    q[t] = qt;
    BFP_UNROLL for (int i = 0; i < W1; ++i) R[i] = (i == 0) ? (tr[0] & qt) : pmux(qt, tr[i], r2[i]);
  }
  w32 rem = 0;
  if constexpr (F::RN) {
    BFP_UNROLL for (int i = 0; i < W1; ++i) rem |= R[i];
  }

  // ez = (ex_eff - lzx) - (ey_eff - lzy) - scale + bias - 1
  w32 ez[EW];
  {
    w32 a[EW], b[EW], la[EW], lb[EW], t1[EW], t2[EW], t3[EW];
    BFP_UNROLL for (int i = 0; i < EW; ++i) {
      a[i] = (i < E) ? X[S + i] : 0u;
      b[i] = (i < E) ? Y[S + i] : 0u;
      la[i] = (i < KN) ? lzx[i] : 0u;
      lb[i] = (i < KN) ? lzy[i] : 0u;
    }
    a[0] |= ~cx.h;
    b[0] |= ~cy.h;
    (void)sub_k<EW>(a, la, t1);   // ex_eff - lzx
    (void)add_k<EW>(t1, lb, 0, t2);  // + lzy
    (void)sub_k<EW>(t2, b, t3);   // - ey_eff
    w32 k[EW];
    constexpr int KB = F::BIAS - 1;  // + bias - 1 (>= 0)
    BFP_UNROLL for (int i = 0; i < EW; ++i) k[i] = ((KB >> i) & 1) ? ONES : 0u;
    w32 t4[EW];
    (void)add_k<EW>(t3, k, 0, t4);
    w32 sc[EW];
    BFP_UNROLL for (int i = 0; i < EW; ++i) sc[i] = i == 0 ? scale : 0u;
    (void)sub_k<EW>(t4, sc, ez);
  }

  w32 Rf[S + 3];
  if constexpr (F::RN) {
    Rf[0] = rem;
    Rf[1] = q[0];
    BFP_UNROLL for (int i = 0; i <= S; ++i) Rf[2 + i] = q[1 + i];
  } else {
    Rf[0] = 0;
    Rf[1] = 0;
    BFP_UNROLL for (int i = 0; i <= S; ++i) Rf[2 + i] = q[i];
  }
  // Special-value rules of bfp_div (arith.hpp:200-205).
  const w32 use_nan = cx.nan | cy.nan | (cx.z & cy.z) | (cx.inf & cy.inf);
  const w32 zero_res = (cx.z | cy.inf) & ~use_nan;
  const w32 inf_res = (cx.inf | cy.z) & ~use_nan;
  finish_round<F, EW>(Rf, ez, sign, zero_res, inf_res, use_nan, Z);
}

// z = round(round(a * b) + c) -- the reference chain bfp_add(bfp_mul(a,b),c),
// fused in registers (config 5).
template <class F>
BFP_HD void mul_add_w(const w32* A, const w32* B, const w32* Cc, w32* Z) {
  w32 p[F::N];
  mul_w<F>(A, B, p);
  add_w<F, false>(p, Cc, Z);
}

// ------------------------------------------------- mul_add: the fast domain
// Most data never touches the subnormal, special-value and overflow machinery
// of the chain, which is 30% of its LUTs (operand normaliser, subnormal-range
// shifter, normaliser budget, Inf / NaN masks, overflow tests).  A unit whose
// 32 elements ALL satisfy, with ea, eb, ec the biased exponent fields,
//   1 <= ea, eb < 3 * 2^(E-2)       a, b finite normals (top two exponent bits
//                                   not both set: magnitudes < 2^(2^(E-2)+1)),
//   2^(E-1) <= ea + eb              the product cannot land below the normal
//                                   range (ez = ea + eb - bias - 1 + top >= 0),
//   ea + eb <= 2^E + 2^(E-1) - 5    nor reach the top two binades: the rounded
//                                   product's field is <= ea + eb - bias + 1
//                                   <= 2^E - 3,
//   2^KN <= ec < 3 * 2^(E-2)        the sum's exponent max(ep, ec) exceeds every
//                                   normalising shift (KN = clog2(S + 5)) and
//                                   max(ep, ec) + 1 <= 2^E - 2 is finite,
// may run mul_add_fast_w: the same network with those signals constant.
// Zeros, subnormals, Inf, NaN, huge or tiny operands fall back to the general
// network.  The kernels evaluate the predicate per unit and vote per warp
// (bfp_kernels.cuh), so a warp takes ONE of the two covers; results are
// identical either way (tests: every triple of 1/4/3 inside the domain, on the
// host and on the GPU, and the GPU sweeps with the fast cover enabled and
// disabled).
template <class F>
constexpr bool mul_add_fast_ok() {
  return F::E > clog2(F::S + 5) && F::E >= 4 && (1 - F::BIAS) <= -F::S - 1;
}

// Lanes of the unit inside the fast domain.
template <class F>
BFP_HD w32 mul_add_fast_domain(const w32* A, const w32* B, const w32* Cc) {
  constexpr int E = F::E, S = F::S, KN = clog2(S + 5);
  const w32* ea = A + S;
  const w32* eb = B + S;
  const w32* ec = Cc + S;
  w32 ha = 0, hb = 0, cbig = 0;
  BFP_UNROLL for (int i = 0; i < E; ++i) {
    ha |= ea[i];
    hb |= eb[i];
  }
  BFP_UNROLL for (int i = KN; i < E; ++i) cbig |= ec[i];
  const w32 small = ~(ea[E - 1] & ea[E - 2]) & ~(eb[E - 1] & eb[E - 2]) & ~(ec[E - 1] & ec[E - 2]);
  // t = ea + eb (E+1 bits): in range iff exactly one of t[E], t[E-1] is set
  // (2^(E-1) <= t < 2^E + 2^(E-1)) and not (t[E-1] = 0 with t[E-2..2] all ones:
  // t >= 2^E + 2^(E-1) - 4)
  w32 t[E + 1];
  t[E] = add_k<E>(ea, eb, 0, t);
  w32 top4 = ~t[E - 1];
  BFP_UNROLL for (int i = 2; i <= E - 2; ++i) top4 &= t[i];
  return ha & hb & cbig & small & (t[E] ^ t[E - 1]) & ~top4;
}

template <class F>
BFP_HD void mul_add_fast_w(const w32* A, const w32* B, const w32* Cc, w32* Z) {
  w32 p[F::N];
  mul_w<F, true>(A, B, p);
  add_w<F, false, true>(p, Cc, Z);
}

}  // namespace bfpg

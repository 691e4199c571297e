// bfp_layout.cuh -- standard <-> bitslice transposition and the scalar codec.
//
// Layout (the memory image of an array of bitfield<lane<1024>>, bitfield.hpp
// :10-28 / pack.hpp:13-15): element i, plane j lives in u32 word
//   ((i >> 10) * N + j) * 32 + ((i >> 5) & 31),  bit (i & 31).
// A "unit" is one 32-element column of a 1024-element block; one thread owns
// one unit, so its N plane words are 128 B apart and a warp's 32 threads
// cover a block with one coalesced 128-B access per plane.
//
// Transposition is a 32x32 bit-matrix transpose held in one thread's
// registers: five commuting exchange stages (16, 8, 4, 2, 1), each swapping
// row-index bit k with column-index bit k (LSB-first indexing: bit c of row r
// <-> bit r of row c).  The reference's transpose64 (pack.hpp:28-39) uses
// MSB-first block swaps on LSB-first data and so computes the anti-diagonal
// transpose; this one is checked against field_from_elements
// / element_of (bitfield.hpp:33-52).  Byte- and half-word stages are done
// with PRMT (__byte_perm) when the encodings are 8 or 16 bits wide.
//
// The codec follows encode_scalar / decode_scalar (format.hpp:101-188) for
// binary32 inputs / outputs.
#pragma once
#if !defined(__CUDACC_RTC__)
#include <string.h>
#endif

#include "bfp_circuits.cuh"

namespace bfpg {

// One exchange stage of distance D over rows [0, R) (R a multiple of 2D).
template <int D, int R>
BFP_HD void xpose_stage(w32* v) {
  constexpr w32 m = D == 16 ? 0x0000ffffu
                  : D == 8  ? 0x00ff00ffu
                  : D == 4  ? 0x0f0f0f0fu
                  : D == 2  ? 0x33333333u
                            : 0x55555555u;
  BFP_UNROLL for (int k = 0; k < R; ++k) {
    if (k & D) continue;
    const w32 a = v[k], b = v[k + D];
    v[k] = (a & m) | ((b << D) & ~m);
    v[k + D] = ((a >> D) & m) | (b & ~m);
  }
}

// Full 32x32 transpose (rows known to be zero fold away at compile time).
BFP_HD void xpose32(w32* v) {
  xpose_stage<16, 32>(v);
  xpose_stage<8, 32>(v);
  xpose_stage<4, 32>(v);
  xpose_stage<2, 32>(v);
  xpose_stage<1, 32>(v);
}

#if defined(__CUDACC__)
BFP_HD w32 prmt(w32 a, w32 b, w32 sel) {
#if defined(__CUDA_ARCH__)
  return __byte_perm(a, b, sel);
#else
  const uint64_t x = (uint64_t(b) << 32) | a;
  w32 r = 0;
  for (int i = 0; i < 4; ++i) r |= w32((x >> (8 * ((sel >> (4 * i)) & 7))) & 0xff) << (8 * i);
  return r;
#endif
}
#else
inline w32 prmt(w32 a, w32 b, w32 sel) {
  const uint64_t x = (uint64_t(b) << 32) | a;
  w32 r = 0;
  for (int i = 0; i < 4; ++i) r |= w32((x >> (8 * ((sel >> (4 * i)) & 7))) & 0xff) << (8 * i);
  return r;
}
#endif

// 32 encodings of <= 8 bits, packed 4 per word (L[q] byte i = element 4q+i)
// -> planes P[0..8).
BFP_HD void enc8_to_planes(const w32* L, w32* P) {
  w32 v[8];
  BFP_UNROLL for (int k = 0; k < 8; ++k) {
    const int q = k >> 2, b = k & 3;
    const w32 sel = w32(b) | (w32(b + 4) << 4);  // byte b of a, byte b of b
    const w32 r1 = prmt(L[q], L[q + 2], sel);      // e_k, e_{k+8}
    const w32 r2 = prmt(L[q + 4], L[q + 6], sel);  // e_{k+16}, e_{k+24}
    v[k] = prmt(r1, r2, 0x5410);
  }
  xpose_stage<4, 8>(v);
  xpose_stage<2, 8>(v);
  xpose_stage<1, 8>(v);
  BFP_UNROLL for (int j = 0; j < 8; ++j) P[j] = v[j];
}

BFP_HD void planes_to_enc8(const w32* P, w32* L) {
  w32 v[8];
  BFP_UNROLL for (int j = 0; j < 8; ++j) v[j] = P[j];
  xpose_stage<1, 8>(v);
  xpose_stage<2, 8>(v);
  xpose_stage<4, 8>(v);
  // v[k] = [e_k, e_{k+8}, e_{k+16}, e_{k+24}]; L[q] = [e_4q .. e_4q+3]
  BFP_UNROLL for (int q = 0; q < 8; ++q) {
    const int k0 = (4 * q) & 7, byte = (4 * q) >> 3;  // element 4q is byte `byte` of v[k0]
    // elements 4q..4q+3 are byte `byte` of v[k0..k0+3]
    const w32 s = w32(byte) | (w32(byte + 4) << 4);
    const w32 r1 = prmt(v[k0], v[k0 + 1], s);
    const w32 r2 = prmt(v[k0 + 2], v[k0 + 3], s);
    L[q] = prmt(r1, r2, 0x5410);
  }
}

// 32 encodings of <= 16 bits, 2 per word (L[q] = e_2q | e_2q+1 << 16)
// -> planes P[0..16).
BFP_HD void enc16_to_planes(const w32* L, w32* P) {
  w32 v[16];
  BFP_UNROLL for (int k = 0; k < 16; ++k) {
    const int q = k >> 1;
    v[k] = (k & 1) ? prmt(L[q], L[q + 8], 0x7632) : prmt(L[q], L[q + 8], 0x5410);
  }
  xpose_stage<8, 16>(v);
  xpose_stage<4, 16>(v);
  xpose_stage<2, 16>(v);
  xpose_stage<1, 16>(v);
  BFP_UNROLL for (int j = 0; j < 16; ++j) P[j] = v[j];
}

BFP_HD void planes_to_enc16(const w32* P, w32* L) {
  w32 v[16];
  BFP_UNROLL for (int j = 0; j < 16; ++j) v[j] = P[j];
  xpose_stage<1, 16>(v);
  xpose_stage<2, 16>(v);
  xpose_stage<4, 16>(v);
  xpose_stage<8, 16>(v);
  // v[k] = e_k | e_{k+16} << 16  (k < 16)
  BFP_UNROLL for (int q = 0; q < 16; ++q) {
    const int k0 = (2 * q) & 15, hi = (2 * q) >> 4;
    L[q] = hi ? prmt(v[k0], v[k0 + 1], 0x7632) : prmt(v[k0], v[k0 + 1], 0x5410);
  }
}

// .bfpraw with a 3-byte stride (pack.hpp:78-109; formats of 17..24 bits):
// 32 records = 96 bytes = 24 words (little-endian) <-> 32 encodings.
BFP_HD void bytes24_to_enc32(const w32* L, w32* V) {
  BFP_UNROLL for (int k = 0; k < 32; ++k) {
    const int b = 3 * k, w = b >> 2, off = b & 3;
    const w32 sel = w32(off) | (w32(off + 1) << 4) | (w32(off + 2) << 8);
    V[k] = prmt(L[w], (w + 1 < 24) ? L[w + 1] : 0u, sel) & 0xffffffu;
  }
}

BFP_HD void enc32_to_bytes24(const w32* V, w32* L) {
  BFP_UNROLL for (int i = 0; i < 24; ++i) {
    // bytes 4i..4i+3 come from records k0 = 4i/3 and k0 + 1
    const int k0 = (4 * i) / 3;
    w32 sel = 0;
    BFP_UNROLL for (int t = 0; t < 4; ++t) {
      const int b = 4 * i + t, k = b / 3, byte = b % 3;
      sel |= w32((k - k0) * 4 + byte) << (4 * t);
    }
    L[i] = prmt(V[k0], (k0 + 1 < 32) ? V[k0 + 1] : 0u, sel);
  }
}

// .bfpraw records of any stride (pack.hpp:78-109): 32 records = 32*ST bytes =
// 8*ST words (little-endian) <-> 32 encodings as (lo, hi) 32-bit halves.
template <int ST>
BFP_HD void bytes_to_enc(const w32* L, w32* lo, w32* hi) {
  constexpr int NW = 8 * ST;
  BFP_UNROLL for (int k = 0; k < 32; ++k) {
    BFP_UNROLL for (int part = 0; part < (ST > 4 ? 2 : 1); ++part) {
      const int b = ST * k + 4 * part;  // first byte of this 32-bit half
      const int nbytes = (ST - 4 * part) < 4 ? (ST - 4 * part) : 4;
      const int w = b >> 2, off = b & 3;
      const w32 sel = w32(off) | (w32(off + 1) << 4) | (w32(off + 2) << 8) | (w32(off + 3) << 12);
      w32 v = prmt(L[w], (w + 1 < NW) ? L[w + 1] : 0u, sel);
      if (nbytes < 4) v &= (1u << (8 * nbytes)) - 1u;
      if (part == 0) lo[k] = v;
      else hi[k] = v;
    }
  }
}

template <int ST>
BFP_HD void enc_to_bytes(const w32* lo, const w32* hi, w32* L) {
  constexpr int NW = 8 * ST;
  BFP_UNROLL for (int i = 0; i < NW; ++i) {
    // bytes 4i..4i+3: byte b belongs to record b / ST, byte (b % ST) of it
    const int r0 = (4 * i) / ST;
    w32 v = 0;
    BFP_UNROLL for (int t = 0; t < 4; ++t) {
      const int b = 4 * i + t, r = b / ST, byte = b % ST;
      const w32 src = (byte < 4) ? lo[r] : hi[r];
      v |= ((src >> (8 * (byte & 3))) & 0xffu) << (8 * t);
    }
    (void)r0;
    L[i] = v;
  }
}

// 32 encodings of <= 32 bits, one per word -> planes (in place).
BFP_HD void enc32_to_planes(w32* v) { xpose32(v); }
BFP_HD void planes_to_enc32(w32* v) { xpose32(v); }

// One unit's element side (8*EB words: EB = 1, 2, 4, 8 device encoding widths,
// 3, 5, 6, 7 .bfpraw strides) <-> its planes (32 words, 64 when EB > 4).
template <int EB>
BFP_HD void elems_to_planes(const w32* L, w32* P /*32 or 64*/) {
  if constexpr (EB == 1) {
    enc8_to_planes(L, P);
  } else if constexpr (EB == 2) {
    enc16_to_planes(L, P);
  } else if constexpr (EB == 4) {
    BFP_UNROLL for (int i = 0; i < 32; ++i) P[i] = L[i];
    enc32_to_planes(P);
  } else if constexpr (EB == 8) {
    BFP_UNROLL for (int k = 0; k < 32; ++k) {
      P[k] = L[2 * k];
      P[32 + k] = L[2 * k + 1];
    }
    enc32_to_planes(P);
    enc32_to_planes(P + 32);
  } else {
    bytes_to_enc<EB>(L, P, P + 32);
    enc32_to_planes(P);
    if constexpr (EB > 4) enc32_to_planes(P + 32);
  }
}

template <int EB>
BFP_HD void planes_to_elems(w32* P /*32 or 64, rows >= N zero*/, w32* L) {
  if constexpr (EB == 1) {
    planes_to_enc8(P, L);
  } else if constexpr (EB == 2) {
    planes_to_enc16(P, L);
  } else if constexpr (EB == 4) {
    planes_to_enc32(P);
    BFP_UNROLL for (int i = 0; i < 32; ++i) L[i] = P[i];
  } else if constexpr (EB == 8) {
    planes_to_enc32(P);
    planes_to_enc32(P + 32);
    BFP_UNROLL for (int k = 0; k < 32; ++k) {
      L[2 * k] = P[k];
      L[2 * k + 1] = P[32 + k];
    }
  } else {
    planes_to_enc32(P);
    if constexpr (EB > 4) planes_to_enc32(P + 32);
    enc_to_bytes<EB>(P, P + 32, L);
  }
}

// ------------------------------------------------------------- codec
// encode_scalar((double)f) for a binary32 input f (format.hpp:125-188):
// correctly rounded, overflow Inf (RN) / max-finite (RZ), FTZ after rounding,
// NaN -> canonical (positive, fraction MSB).
template <class F>
BFP_HD w32 encode_f32(w32 u) {
  constexpr int E = F::E, S = F::S;
  constexpr int EMIN = 1 - F::BIAS, EMAX = F::BIAS;
  constexpr w32 EMASK = (1u << E) - 1;
  const w32 sign = (u >> 31) << (E + S);
  const w32 a = u & 0x7fffffffu;
  if (a >= 0x7f800000u) {
    if (a > 0x7f800000u) return (EMASK << S) | (1u << (S - 1));
    return sign | (EMASK << S);
  }
  if (a == 0) return sign;
  const int ef = int(a >> 23);
  const w32 sig = ef ? ((a & 0x7fffffu) | 0x800000u) : a;
  const int exp2 = (ef ? ef : 1) - 150;  // value = sig * 2^exp2
#if defined(__CUDA_ARCH__)
  const int msb = 31 - __clz(sig);
#else
  const int msb = 31 - __builtin_clz(sig);
#endif
  const int unb = exp2 + msb;
  const int ulp_exp = (unb >= EMIN ? unb : EMIN) - S;
  const int shift = ulp_exp - exp2;
  uint64_t kept;
  w32 guard = 0, sticky = 0;
  if (shift <= 0) {
    kept = uint64_t(sig) << (-shift);
  } else if (shift > 32) {
    kept = 0;
    sticky = 1;
  } else {
    kept = shift == 32 ? 0 : (sig >> shift);
    guard = (sig >> (shift - 1)) & 1u;
    sticky = (shift > 1) ? ((sig & ((1u << (shift - 1)) - 1u)) != 0) : 0u;
  }
  if (F::RN && guard && (sticky || (kept & 1u))) ++kept;
  int res_exp = ulp_exp + S;
  if (kept >= (uint64_t(2) << S)) {
    kept >>= 1;
    ++res_exp;
  }
  if (kept == 0) return sign;
  if (kept < (uint64_t(1) << S)) {
    if (F::FTZ) return sign;
    return sign | w32(kept);
  }
  if (res_exp > EMAX) {
    if (F::RN) return sign | (EMASK << S);
    return sign | ((EMASK - 1) << S) | ((1u << S) - 1u);
  }
  return sign | (w32(res_exp + F::BIAS) << S) | (w32(kept) & ((1u << S) - 1u));
}

// (float)decode_scalar(enc) as binary32 bits (format.hpp:101-123); every
// value of a format with E <= 8, S <= 23 is exact in binary32.  NaN ->
// quiet_NaN() -> 0x7fc00000.
template <class F>
BFP_HD w32 decode_f32(w32 enc) {
  constexpr int E = F::E, S = F::S;
  constexpr w32 EMASK = (1u << E) - 1;
  const w32 sign = ((enc >> (E + S)) & 1u) << 31;
  const w32 be = (enc >> S) & EMASK;
  const w32 fr = enc & ((1u << S) - 1u);
  if (be == EMASK) return fr ? 0x7fc00000u : (sign | 0x7f800000u);
  if (be == 0) {
    if (fr == 0) return sign;
#if defined(__CUDA_ARCH__)
    const int p = 31 - __clz(fr);
#else
    const int p = 31 - __builtin_clz(fr);
#endif
    const int fexp = p + (1 - F::BIAS) - S + 127;  // biased binary32 exponent
    constexpr int SUBSH = (1 - F::BIAS) - S + 149;  // binary32-subnormal placement
    if constexpr (SUBSH < 32) {
      if (fexp < 1) return sign | (fr << SUBSH);
    }
    return sign | (w32(fexp) << 23) | ((fr << (23 - p)) & 0x7fffffu);
  }
  return sign | (w32(int(be) - F::BIAS + 127) << 23) | (fr << (23 - S));
}

// ------------------------------------------------ branch-free codec
// The kernels use these; encode_f32 / decode_f32 above are the direct
// restatements they are checked against (tests/test_circuits_host.py).

// Subnormal-range rounding: frac = round(|x| / 2^(emin - S)) for |x| < 2^emin.
template <class F>
BFP_HD w32 sub_round(w32 a) {
  constexpr int EMIN = 1 - F::BIAS, S = F::S;
#if defined(__CUDA_ARCH__)
  // one FADD at the subnormal ulp: |x| + 2^(emin - S + 23) rounds |x| to a
  // multiple of 2^(emin - S) (RN-even or RZ in hardware, exactly like the
  // reference's guard/sticky rounding); the sum's low bits are the fraction.
  const float M = __uint_as_float(w32(127 + EMIN - S + 23) << 23);
  const float x = __uint_as_float(a);
  const float sum = F::RN ? __fadd_rn(x, M) : __fadd_rz(x, M);
  return __float_as_uint(sum) - __float_as_uint(M);
#else
  const int ef = int(a >> 23);
  const uint64_t sig = ef ? ((a & 0x7fffffu) | 0x800000u) : a;
  const int e = (ef ? ef : 1) - 150;
  const int shift = (EMIN - S) - e;  // >= 1 in the subnormal range
  if (shift >= 40) return 0;
  uint64_t kept = sig >> shift;
  const uint64_t g = (sig >> (shift - 1)) & 1u;
  const uint64_t st = (sig & ((uint64_t(1) << (shift - 1)) - 1)) != 0;
  if (F::RN && g && (st || (kept & 1u))) ++kept;
  return w32(kept);
#endif
}

template <class F>
BFP_HD w32 encode_f32_fast(w32 u) {
  constexpr int E = F::E, S = F::S, SH = 23 - S;
  constexpr int EMIN = 1 - F::BIAS, EMAX = F::BIAS;
  constexpr w32 EMASK = (1u << E) - 1;
  constexpr w32 FMASK = (1u << S) - 1;
  const w32 a = u & 0x7fffffffu;
  w32 t = a;
  if constexpr (SH > 0 && F::RN) t = a + ((1u << (SH - 1)) - 1u) + ((a >> SH) & 1u);
  const w32 enc_n = (t >> SH) - (w32(127 - F::BIAS) << S);
  constexpr w32 MINN = w32(127 + EMIN) << 23;     // 2^emin
  constexpr w32 OVF = w32(127 + EMAX + 1) << 23;  // 2^(emax+1)
  w32 r = (a < MINN) ? sub_round<F>(a) : enc_n;
  if constexpr (OVF < 0x7f800000u || F::RN) {
    if (t >= OVF) r = F::RN ? (EMASK << S) : (((EMASK - 1) << S) | FMASK);
  }
  if constexpr (F::FTZ) r = (r <= FMASK) ? 0u : r;
  r = (a == 0x7f800000u) ? (EMASK << S) : r;
  r |= (u >> 31) << (E + S);
  return (a > 0x7f800000u) ? ((EMASK << S) | (1u << (S - 1))) : r;
}

template <class F>
BFP_HD w32 decode_f32_fast(w32 enc) {
  constexpr int E = F::E, S = F::S, SH = 23 - S;
  constexpr int EMIN = 1 - F::BIAS;
  constexpr w32 EMASK = (1u << E) - 1;
  const w32 mag = enc & ((1u << (E + S)) - 1u);
  const w32 be = mag >> S;
  const w32 r_n = (mag << SH) + (w32(127 - F::BIAS) << 23);
  // subnormal: as_float(bits(M) + frac) - M == frac * 2^(emin - S), exact
  constexpr w32 MB = w32(127 + EMIN - S + 23) << 23;
#if defined(__CUDA_ARCH__)
  const w32 r_s = __float_as_uint(__uint_as_float(MB + mag) - __uint_as_float(MB));
#else
  float fa, fm;
  const w32 ta = MB + mag, tm = MB;
  memcpy(&fa, &ta, 4);
  memcpy(&fm, &tm, 4);
  const float d = fa - fm;
  w32 r_s;
  memcpy(&r_s, &d, 4);
#endif
  w32 r = (be == 0) ? r_s : r_n;
  r = (be == EMASK) ? 0x7f800000u : r;
  r |= ((enc >> (E + S)) & 1u) << 31;
  return (be == EMASK && (mag & ((1u << S) - 1u))) ? 0x7fc00000u : r;
}

// ------------------------------------------------------ binary64 codec
// encode_scalar(double) / decode_scalar -> double, format.hpp:101-188, for
// any legal format (n <= 64): the reference converter restated on 64-bit
// integers (decode is exact: every finite value of a legal format is a
// binary64 value).
BFP_HD int clz64(uint64_t v) {
#if defined(__CUDA_ARCH__)
  return __clzll(static_cast<long long>(v));
#else
  return v ? __builtin_clzll(v) : 64;
#endif
}

template <class F>
BFP_HD uint64_t encode_f64(uint64_t bits) {
  constexpr int E = F::E, S = F::S;
  constexpr int EMIN = 1 - F::BIAS, EMAX = F::BIAS;
  constexpr uint64_t EMASK = (uint64_t(1) << E) - 1;
  constexpr uint64_t FMASK = (uint64_t(1) << S) - 1;
  const uint64_t sign = (bits >> 63) << (E + S);
  const uint64_t e64 = (bits >> 52) & 0x7ff, f64 = bits & ((uint64_t(1) << 52) - 1);
  if (e64 == 0x7ff) return f64 ? ((EMASK << S) | (uint64_t(1) << (S - 1))) : (sign | (EMASK << S));
  if (e64 == 0 && f64 == 0) return sign;
  const uint64_t sig = e64 ? ((uint64_t(1) << 52) | f64) : f64;
  const int exp2 = e64 ? int(e64) - 1075 : -1074;
  const int unb = exp2 + (63 - clz64(sig));
  const int ulp_exp = (unb >= EMIN ? unb : EMIN) - S;
  const int shift = ulp_exp - exp2;
  uint64_t kept;
  bool guard = false, sticky = false;
  if (shift <= 0) {
    kept = sig << (-shift);
  } else if (shift > 64) {
    kept = 0;
    sticky = true;
  } else {
    kept = shift == 64 ? 0 : (sig >> shift);
    guard = (sig >> (shift - 1)) & 1u;
    if (shift > 1) sticky = (sig & ((uint64_t(1) << (shift - 1)) - 1)) != 0;
  }
  if (F::RN && guard && (sticky || (kept & 1u))) ++kept;
  int res_exp = ulp_exp + S;
  if (S < 63 && kept >= (uint64_t(2) << S)) {
    kept >>= 1;
    ++res_exp;
  }
  if (kept == 0) return sign;
  if (kept < (uint64_t(1) << S)) return F::FTZ ? sign : (sign | kept);
  if (res_exp > EMAX) return F::RN ? (sign | (EMASK << S)) : (sign | ((EMASK - 1) << S) | FMASK);
  return sign | (uint64_t(res_exp + F::BIAS) << S) | (kept & FMASK);
}

template <class F>
BFP_HD uint64_t decode_f64(uint64_t enc) {
  constexpr int E = F::E, S = F::S;
  constexpr int EMIN = 1 - F::BIAS;
  constexpr uint64_t EMASK = (uint64_t(1) << E) - 1;
  constexpr uint64_t FMASK = (uint64_t(1) << S) - 1;
  const uint64_t sign = ((enc >> (E + S)) & 1u) << 63;
  const uint64_t be = (enc >> S) & EMASK, fr = enc & FMASK;
  if (be == EMASK) return fr ? 0x7ff8000000000000ull : (sign | 0x7ff0000000000000ull);
  if (be == 0) {
    if (fr == 0) return sign;
    const int p = 63 - clz64(fr);
    const int dexp = p + EMIN - S;  // unbiased exponent of the leading bit
    if constexpr (EMIN - S < -1022) {  // binary64 subnormals occur (e = 11 formats)
      if (dexp < -1022) return sign | (fr << (EMIN - S + 1074));
    }
    return sign | (uint64_t(dexp + 1023) << 52) | ((fr << (52 - p)) & ((uint64_t(1) << 52) - 1));
  }
  return sign | (uint64_t(int(be) - F::BIAS + 1023) << 52) | (fr << (52 - S));
}

// Canonical NaN in the bitslice domain: every element whose exponent planes
// are all ones and whose fraction is nonzero becomes the canonical NaN
// (positive, fraction MSB only -- format.hpp:49-52).  ~(E+S)/2 + N LOP3s
// per 32 elements.
template <class F>
BFP_HD void canon_nan_planes(w32* P) {
  constexpr int E = F::E, S = F::S;
  w32 ea = ONES, fo = 0;
  BFP_UNROLL for (int i = 0; i < E; ++i) ea &= P[S + i];
  BFP_UNROLL for (int i = 0; i < S; ++i) fo |= P[i];
  const w32 nan = ea & fo;
  BFP_UNROLL for (int j = 0; j < S - 1; ++j) P[j] &= ~nan;
  P[S - 1] |= nan;
  P[S + E] &= ~nan;
}

// Hardware conversion applies when IEEE binary16 / bfloat16 conversion
// equals encode_scalar / decode_scalar for the format (RN-even or RZ,
// gradual underflow, overflow to Inf / max-finite) -- NaN aside, which the
// planes fix above canonicalises.  0 = generic, 1 = binary16, 2 = bfloat16.
template <class F>
struct HwCodec {
  // FTZ formats too: encode_scalar flushes AFTER rounding (format.hpp:173-177),
  // so the hardware conversion followed by a flush of subnormal results is
  // exact (floats_to_planes), and decode_scalar has no DAZ (format.hpp:114-116).
  static constexpr int kind = (F::E == 5 && F::S == 10) ? 1 : (F::E == 8 && F::S == 7) ? 2 : 0;
};

#if defined(__CUDACC__)
// two floats -> two encodings packed lo | hi << 16 (cvt.*.x2: first source
// to the upper half)
template <int KIND, bool RN>
__device__ __forceinline__ w32 hw_cvt2(float lo, float hi) {
  w32 r;
  if constexpr (KIND == 1) {
    if constexpr (RN) asm("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    else asm("cvt.rz.f16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  } else {
    if constexpr (RN) asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    else asm("cvt.rz.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  }
  return r;
}

template <int KIND>
__device__ __forceinline__ w32 hw_widen(w32 h16) {
  if constexpr (KIND == 1) {
    float f;
    asm("{.reg .b16 h; cvt.u16.u32 h, %1; cvt.f32.f16 %0, h;}" : "=f"(f) : "r"(h16));
    // NaN inputs are canonical and positive here (canon_nan_planes); the
    // widening may return its own canonical NaN (0x7fffffff): a signed min
    // maps every positive NaN pattern above 0x7fc00000 to quiet_NaN() and
    // leaves finite values, +Inf and all negative values unchanged.
    return w32(min(int(__float_as_uint(f)), 0x7fc00000));
  } else {
    return h16 << 16;
  }
}
#endif

}  // namespace bfpg

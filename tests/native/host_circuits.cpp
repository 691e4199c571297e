// tests/native/host_circuits.cpp -- TEST HARNESS ONLY.
// Compiles the device networks, transposes and codec
// (paper_1602_04716_b200/csrc/bfp_circuits.cuh, bfp_layout.cuh) for the host
// so tests can check them exhaustively against the oracle without a GPU.
// Operands use the device plane layout.
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <utility>

#include "../../paper_1602_04716_b200/csrc/bfp_circuits.cuh"
#include "../../paper_1602_04716_b200/csrc/bfp_formats.h"
#include "../../paper_1602_04716_b200/csrc/bfp_layout.cuh"
// the generated LOP3 covers (paper_1602_04716_b200/build.py writes them)
#include "../../paper_1602_04716_b200/csrc/gen/gen_3_2.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_4_3.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_5_3.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_5_7.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_5_10.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_6_9.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_8_7.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_8_15.cuh"
#include "../../paper_1602_04716_b200/csrc/gen/gen_8_23.cuh"

using namespace bfpg;

template <class F>
static void run(int op, const uint32_t* x, const uint32_t* y, const uint32_t* c, uint32_t* z,
                size_t nblocks) {
  constexpr int N = F::N;
  for (size_t b = 0; b < nblocks; ++b)
    for (int t = 0; t < 32; ++t) {
      w32 X[N], Y[N], C[N], Z[N];
      for (int j = 0; j < N; ++j) {
        const size_t w = (b * N + j) * 32 + t;
        X[j] = x[w];
        Y[j] = y[w];
        C[j] = c ? c[w] : 0u;
      }
      switch (op) {
        case 10: Gen<F, 0>::run(X, Y, C, Z); break;  // generated covers
        case 11: Gen<F, 1>::run(X, Y, C, Z); break;
        case 12: Gen<F, 2>::run(X, Y, C, Z); break;
        case 13: Gen<F, 3>::run(X, Y, C, Z); break;
        case 14: Gen<F, 4>::run(X, Y, C, Z); break;
        case 0: add_w<F, false>(X, Y, Z); break;
        case 1: add_w<F, true>(X, Y, Z); break;
        case 2: mul_w<F>(X, Y, Z); break;
        case 3: div_w<F>(X, Y, Z); break;
        case 4: mul_add_w<F>(X, Y, C, Z); break;
        // mul_add on its fast domain: template, generated cover, and the
        // domain predicate itself (plane 0 = lanes inside the domain)
        case 5:
          if constexpr (mul_add_fast_ok<F>()) mul_add_fast_w<F>(X, Y, C, Z);
          else return;
          break;
        case 15:
          if constexpr (Gen<F, 5>::ok) Gen<F, 5>::run(X, Y, C, Z);
          else return;
          break;
        case 6:
          if constexpr (mul_add_fast_ok<F>()) {
            for (int j = 0; j < N; ++j) Z[j] = 0;
            Z[0] = mul_add_fast_domain<F>(X, Y, C);
          } else {
            return;
          }
          break;
        default: return;
      }
      for (int j = 0; j < N; ++j) z[(b * N + j) * 32 + t] = Z[j];
    }
}

template <class F>
static void codec(int dir, const uint32_t* in, uint32_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) {
    switch (dir) {
      case 0: out[i] = encode_f32<F>(in[i]); break;
      case 1: out[i] = decode_f32<F>(in[i]); break;
      case 2: out[i] = encode_f32_fast<F>(in[i]); break;
      default: out[i] = decode_f32_fast<F>(in[i]); break;
    }
  }
}

template <int E_, int S_, class Fn>
static void with_fmt(int rn, int ftz, Fn&& fn) {
  if (rn && !ftz) fn(Format<E_, S_, true, false>{});
  if (rn && ftz) fn(Format<E_, S_, true, true>{});
  if (!rn && !ftz) fn(Format<E_, S_, false, false>{});
  if (!rn && ftz) fn(Format<E_, S_, false, true>{});
}

template <class Fn>
static int dispatch(unsigned e, unsigned s, int rn, int ftz, Fn&& fn) {
#define DISPATCH(E_, S_)                   \
  if (e == E_ && s == S_) {                \
    with_fmt<E_, S_>(rn, ftz, fn);         \
    return 0;                              \
  }
  BFP_FORMAT_LIST(DISPATCH)
#undef DISPATCH
  return 4;
}

extern "C" int host_binop(int op, unsigned e, unsigned s, int rn, int ftz, const uint32_t* x,
                          const uint32_t* y, const uint32_t* c, uint32_t* z, size_t nblocks) {
  return dispatch(e, s, rn, ftz, [&](auto f) { run<decltype(f)>(op, x, y, c, z, nblocks); });
}

// dir 0: float32 bits -> encoding (encode_f32); dir 1: encoding -> float32 bits.
extern "C" int host_codec(int dir, unsigned e, unsigned s, int rn, int ftz, const uint32_t* in,
                          uint32_t* out, size_t n) {
  return dispatch(e, s, rn, ftz, [&](auto f) { codec<decltype(f)>(dir, in, out, n); });
}

// Encodings / .bfpraw records (eb = 1..8 bytes each) <-> planes of nbits
// planes, through the same register transposes the kernels use (tail zero).
template <int EB>
static void pack_t(unsigned nbits, const uint8_t* enc, size_t n, uint32_t* planes) {
  const size_t blocks = (n + 1023) / 1024;
  for (size_t u = 0; u < blocks * 32; ++u) {
    w32 L[8 * EB] = {0};
    for (int b = 0; b < 32 * EB; ++b) {
      const size_t i = u * 32 + size_t(b / EB);
      if (i < n) L[b >> 2] |= w32(enc[u * 32 * EB + b]) << (8 * (b & 3));
    }
    w32 P[EB > 4 ? 64 : 32];
    elems_to_planes<EB>(L, P);
    for (unsigned j = 0; j < nbits; ++j) planes[((u >> 5) * nbits + j) * 32 + (u & 31)] = P[j];
  }
}

template <int EB>
static void unpack_t(unsigned nbits, const uint32_t* planes, size_t n, uint8_t* enc) {
  const size_t units = (n + 31) / 32;
  for (size_t u = 0; u < units; ++u) {
    w32 P[EB > 4 ? 64 : 32] = {0};
    for (unsigned j = 0; j < nbits; ++j) P[j] = planes[((u >> 5) * nbits + j) * 32 + (u & 31)];
    w32 L[8 * EB];
    planes_to_elems<EB>(P, L);
    for (int b = 0; b < 32 * EB; ++b) {
      const size_t i = u * 32 + size_t(b / EB);
      if (i < n) enc[u * 32 * EB + b] = uint8_t(L[b >> 2] >> (8 * (b & 3)));
    }
  }
}

extern "C" int host_pack_enc(int eb, unsigned nbits, const uint8_t* enc, size_t n,
                             uint32_t* planes) {
  switch (eb) {
    case 1: pack_t<1>(nbits, enc, n, planes); break;
    case 2: pack_t<2>(nbits, enc, n, planes); break;
    case 3: pack_t<3>(nbits, enc, n, planes); break;
    case 4: pack_t<4>(nbits, enc, n, planes); break;
    case 5: pack_t<5>(nbits, enc, n, planes); break;
    case 6: pack_t<6>(nbits, enc, n, planes); break;
    case 7: pack_t<7>(nbits, enc, n, planes); break;
    case 8: pack_t<8>(nbits, enc, n, planes); break;
    default: return 1;
  }
  return 0;
}

extern "C" int host_unpack_enc(int eb, unsigned nbits, const uint32_t* planes, size_t n,
                               uint8_t* enc) {
  switch (eb) {
    case 1: unpack_t<1>(nbits, planes, n, enc); break;
    case 2: unpack_t<2>(nbits, planes, n, enc); break;
    case 3: unpack_t<3>(nbits, planes, n, enc); break;
    case 4: unpack_t<4>(nbits, planes, n, enc); break;
    case 5: unpack_t<5>(nbits, planes, n, enc); break;
    case 6: unpack_t<6>(nbits, planes, n, enc); break;
    case 7: unpack_t<7>(nbits, planes, n, enc); break;
    case 8: unpack_t<8>(nbits, planes, n, enc); break;
    default: return 1;
  }
  return 0;
}

// 96 .bfpraw bytes (32 records of 3 bytes) -> 32 encodings -> 96 bytes.
extern "C" int host_raw3(const uint8_t* bytes96, uint32_t* enc32, uint8_t* back96) {
  w32 L[24], V[32], B[24];
  std::memcpy(L, bytes96, 96);
  bytes24_to_enc32(L, V);
  std::memcpy(enc32, V, 128);
  enc32_to_bytes24(V, B);
  std::memcpy(back96, B, 96);
  return 0;
}

// binary64 codec (encode_f64 / decode_f64) on u64 bit patterns: dir 0 encode,
// 1 decode; the listed formats plus a few wide ones (n up to 64).
template <class F>
static void codec64(int dir, const uint64_t* in, uint64_t* out, size_t n) {
  for (size_t i = 0; i < n; ++i) out[i] = dir == 0 ? encode_f64<F>(in[i]) : decode_f64<F>(in[i]);
}

extern "C" int host_codec64(int dir, unsigned e, unsigned s, int rn, int ftz, const uint64_t* in,
                            uint64_t* out, size_t n) {
  auto fn = [&](auto f) { codec64<decltype(f)>(dir, in, out, n); };
  if (e == 11 && s == 52) { with_fmt<11, 52>(rn, ftz, fn); return 0; }
  if (e == 10 && s == 40) { with_fmt<10, 40>(rn, ftz, fn); return 0; }
  if (e == 11 && s == 20) { with_fmt<11, 20>(rn, ftz, fn); return 0; }
  if (e == 2 && s == 1) { with_fmt<2, 1>(rn, ftz, fn); return 0; }
  return dispatch(e, s, rn, ftz, fn);
}

// Significand products (tests only): which = 0 array (sig_product), 1 Booth
// (sig_product_booth).  a, b: S+1 words each, p: 2S+2 words.
template <int S>
static void product_t(int which, const uint32_t* a, const uint32_t* b, uint32_t* p) {
  if (which == 0)
    bfpg::sig_product<S>(a, b, p);
  else
    bfpg::sig_product_booth<S>(a, b, p);
}
template <int... Ks>
static int product_dispatch(int s, int which, const uint32_t* a, const uint32_t* b, uint32_t* p,
                            std::integer_sequence<int, Ks...>) {
  int ok = -1;  // S = K + 2, 2..30
  ((s == Ks + 2 ? (product_t<Ks + 2>(which, a, b, p), ok = 0) : 0), ...);
  return ok;
}
extern "C" int host_product(int s, int which, const uint32_t* a, const uint32_t* b, uint32_t* p) {
  return product_dispatch(s, which, a, b, p, std::make_integer_sequence<int, 29>{});
}

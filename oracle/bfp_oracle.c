/* oracle/bfp_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the
 * product).  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load the library built from this file (oracle/liboracle.so).
 *
 * A plain-C, value-level restatement of the reference's bitslice FP path:
 *
 *   orc_encode   <- encode_scalar   format.hpp:125-188 (binary64 -> format)
 *   orc_decode   <- decode_scalar   format.hpp:101-123 (format -> binary64)
 *   orc_add/sub/mul/div/mul_add <- bfp_add/bfp_sub/bfp_mul/bfp_div
 *                                   (arith.hpp:235-444), restated by value:
 *       decode both operands exactly, combine them in binary64 under
 *       fesetround(FE_TONEAREST | FE_TOWARDZERO), encode the result.
 *       This is exact-then-rounded for every format with s <= 24:
 *         - products of two (s+1)-bit significands are exact in binary64;
 *         - RN double rounding is innocuous since 53 >= 2(s+1)+2;
 *         - RZ truncation composes with RZ truncation.
 *       The IEEE conventions of the circuits are all carried by encode /
 *       binary64: canonical positive NaN (format.hpp:49-52), +0 from exact
 *       cancellation and -0 only for (-0)+(-0) (arith.hpp:312-316), overflow
 *       to Inf under RN / max-finite under RZ (arith.hpp:143-146), FTZ after
 *       rounding with no input DAZ (arith.hpp:135-141).
 *   orc_pack_planes / orc_unpack_planes <- field_from_elements / element_of
 *       (bitfield.hpp:33-52): element i, plane j -> u32 word
 *       ((i>>10)*n + j)*32 + ((i>>5)&31), bit i&31.
 *
 * Parity pin: tests/test_oracle.py checks this file against the reference
 * headers compiled in place (oracle/_ref, see oracle/Makefile) exhaustively
 * for the <= 9-bit formats and on seeded random + directed operands for the
 * rest, and against the golden fixtures in tests/golden/.
 *
 * Build: gcc -O2 -std=c11 -frounding-math -ffp-contract=off -fPIC -shared.
 */
#include <fenv.h>
#include <math.h>
#include <stddef.h>
#include <stdint.h>
#include <string.h>

#pragma STDC FENV_ACCESS ON

typedef struct {
  unsigned e, s;
  int rn, ftz;
} orc_fmt;

static uint64_t make_enc(const orc_fmt* f, unsigned sign, uint64_t bexp, uint64_t frac) {
  return ((uint64_t)(sign & 1u) << (f->e + f->s)) | (bexp << f->s) | frac;
}
static uint64_t exp_field_max(const orc_fmt* f) { return (1ull << f->e) - 1; }
static int bias_of(const orc_fmt* f) { return (1 << (f->e - 1)) - 1; }

static int clz64(uint64_t v) { return v ? __builtin_clzll(v) : 64; }

/* encode_scalar, format.hpp:125-188 */
uint64_t orc_encode(double x, unsigned e, unsigned s, int rn, int ftz) {
  orc_fmt F = {e, s, rn, ftz};
  const orc_fmt* f = &F;
  uint64_t bits;
  memcpy(&bits, &x, sizeof bits);
  const unsigned sign = (unsigned)(bits >> 63);
  const uint64_t e64 = (bits >> 52) & 0x7ff;
  const uint64_t f64 = bits & ((1ull << 52) - 1);
  if (e64 == 0x7ff) {
    if (f64) return make_enc(f, 0, exp_field_max(f), 1ull << (s - 1)); /* canonical NaN */
    return make_enc(f, sign, exp_field_max(f), 0);                      /* Inf */
  }
  if (e64 == 0 && f64 == 0) return make_enc(f, sign, 0, 0);
  const uint64_t sig = e64 ? ((1ull << 52) | f64) : f64;
  const int exp2 = e64 ? (int)e64 - 1023 - 52 : -1022 - 52;
  const int msb = 63 - clz64(sig);
  const int unb = exp2 + msb; /* floor(log2|x|) */
  const int emin = 1 - bias_of(f), emax = bias_of(f);
  const int ulp_exp = (unb >= emin ? unb : emin) - (int)s;
  const int shift = ulp_exp - exp2;
  uint64_t kept;
  int guard = 0, sticky = 0;
  if (shift <= 0) {
    kept = sig << -shift;
  } else if (shift > 64) {
    kept = 0;
    sticky = 1;
  } else {
    kept = shift == 64 ? 0 : sig >> shift;
    guard = (int)((sig >> (shift - 1)) & 1u);
    if (shift > 1) sticky = (sig & ((1ull << (shift - 1)) - 1)) != 0;
  }
  if (rn && guard && (sticky || (kept & 1u))) ++kept;
  int res_exp = ulp_exp + (int)s;
  if (kept >= (2ull << s)) {
    kept >>= 1;
    ++res_exp;
  }
  if (kept == 0) return make_enc(f, sign, 0, 0);
  if (kept < (1ull << s)) {
    if (ftz) return make_enc(f, sign, 0, 0);
    return make_enc(f, sign, 0, kept);
  }
  if (res_exp > emax)
    return rn ? make_enc(f, sign, exp_field_max(f), 0)
              : make_enc(f, sign, exp_field_max(f) - 1, (1ull << s) - 1);
  return make_enc(f, sign, (uint64_t)(res_exp + bias_of(f)), kept & ((1ull << s) - 1));
}

/* decode_scalar, format.hpp:101-123 (exact: every finite value of a legal
 * format is a binary64 value) */
double orc_decode(uint64_t enc, unsigned e, unsigned s) {
  orc_fmt F = {e, s, 1, 0};
  const orc_fmt* f = &F;
  const unsigned sign = (unsigned)((enc >> (e + s)) & 1u);
  const uint64_t bexp = (enc >> s) & exp_field_max(f);
  const uint64_t frac = enc & ((1ull << s) - 1);
  const double sg = sign ? -1.0 : 1.0;
  if (bexp == exp_field_max(f)) return frac ? NAN : sg * INFINITY;
  if (bexp == 0) {
    if (!frac) return sg * 0.0;
    return sg * ldexp((double)frac, 1 - bias_of(f) - (int)s);
  }
  return sg * ldexp((double)((1ull << s) | frac), (int)bexp - bias_of(f) - (int)s);
}

enum { ORC_ADD = 0, ORC_SUB = 1, ORC_MUL = 2, ORC_DIV = 3, ORC_MUL_ADD = 4 };

static double rounded_op(int op, double a, double b, int rn) {
  volatile double va = a, vb = b, r;
  const int want = rn ? FE_TONEAREST : FE_TOWARDZERO;
  const int old = fegetround();
  if (old != want) fesetround(want);
  switch (op) {
    case ORC_ADD: r = va + vb; break;
    case ORC_SUB: r = va - vb; break;
    case ORC_MUL: r = va * vb; break;
    default: r = va / vb; break;
  }
  if (old != want) fesetround(old);
  return r;
}

/* Value-level bfp_add / bfp_sub / bfp_mul / bfp_div (arith.hpp:235-444). */
uint64_t orc_binop(int op, unsigned e, unsigned s, int rn, int ftz, uint64_t x, uint64_t y) {
  const double a = orc_decode(x, e, s), b = orc_decode(y, e, s);
  return orc_encode(rounded_op(op, a, b, rn), e, s, rn, ftz);
}

/* The chain bfp_add(bfp_mul(a, b), c): two roundings. */
uint64_t orc_mul_add(unsigned e, unsigned s, int rn, int ftz, uint64_t a, uint64_t b, uint64_t c) {
  const uint64_t p = orc_binop(ORC_MUL, e, s, rn, ftz, a, b);
  return orc_binop(ORC_ADD, e, s, rn, ftz, p, c);
}

/* field_from_elements (bitfield.hpp:33-43), one 1024-element block at a time;
 * the tail of the last block is zero-filled like pack.hpp:50. */
void orc_pack_planes(const uint64_t* enc, size_t n, uint32_t* planes, unsigned nbits) {
  const size_t blocks = (n + 1023) / 1024;
  memset(planes, 0, blocks * nbits * 128);
  for (size_t i = 0; i < n; ++i) {
    const size_t blk = i >> 10;
    const unsigned w = (unsigned)((i >> 5) & 31), bit = (unsigned)(i & 31);
    for (unsigned j = 0; j < nbits; ++j)
      planes[(blk * nbits + j) * 32 + w] |= (uint32_t)((enc[i] >> j) & 1u) << bit;
  }
}

/* element_of (bitfield.hpp:45-52) */
void orc_unpack_planes(const uint32_t* planes, size_t n, uint64_t* enc, unsigned nbits) {
  for (size_t i = 0; i < n; ++i) {
    const size_t blk = i >> 10;
    const unsigned w = (unsigned)((i >> 5) & 31), bit = (unsigned)(i & 31);
    uint64_t v = 0;
    for (unsigned j = 0; j < nbits; ++j)
      v |= (uint64_t)((planes[(blk * nbits + j) * 32 + w] >> bit) & 1u) << j;
    enc[i] = v;
  }
}

/* Array forms over encodings (u64 per element). */
void orc_binop_array(int op, unsigned e, unsigned s, int rn, int ftz, const uint64_t* x,
                     const uint64_t* y, const uint64_t* c, uint64_t* z, size_t n) {
  if (op == ORC_MUL_ADD) {
    for (size_t i = 0; i < n; ++i) z[i] = orc_mul_add(e, s, rn, ftz, x[i], y[i], c[i]);
  } else {
    for (size_t i = 0; i < n; ++i) z[i] = orc_binop(op, e, s, rn, ftz, x[i], y[i]);
  }
}

void orc_encode_f32_array(const float* in, size_t n, uint64_t* out, unsigned e, unsigned s,
                          int rn, int ftz) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_encode((double)in[i], e, s, rn, ftz);
}

void orc_decode_f32_array(const uint64_t* enc, size_t n, float* out, unsigned e, unsigned s) {
  for (size_t i = 0; i < n; ++i) out[i] = (float)orc_decode(enc[i], e, s);
}

/* All (x, y) pairs of an n-bit format in row-major order: z[x * 2^n + y]. */
void orc_binop_exhaustive(int op, unsigned e, unsigned s, int rn, int ftz, uint64_t* z) {
  const uint64_t cnt = 1ull << (1 + e + s);
  for (uint64_t x = 0; x < cnt; ++x)
    for (uint64_t y = 0; y < cnt; ++y) z[x * cnt + y] = orc_binop(op, e, s, rn, ftz, x, y);
}

/* binary64 array forms of encode_scalar / decode_scalar (format.hpp:101-188) */
void orc_encode_f64_array(const double* in, size_t n, uint64_t* out, unsigned e, unsigned s,
                          int rn, int ftz) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_encode(in[i], e, s, rn, ftz);
}

void orc_decode_f64_array(const uint64_t* enc, size_t n, double* out, unsigned e, unsigned s) {
  for (size_t i = 0; i < n; ++i) out[i] = orc_decode(enc[i], e, s);
}

/* ------------------------------------------------------------------------
 * Full-size verification (tests only): the oracle's expected result of every
 * element, compared with the device's output, on all host threads.
 *
 * orc_verify: op 0..4 = add/sub/mul/div/mul_add, 5 = pack (the encoding of a
 * itself), 6 = unpack to float32 ((float)decode(encode(a))).  Inputs a, b, c
 * are u32 encodings (in_kind 0) or float32 values through encode_scalar
 * (in_kind 1), element i at index i.  got = the device planes
 * (field_from_elements image, bitfield.hpp:33-52) for ops 0..5, float32 bits
 * for op 6.  Returns the number of mismatching elements; the first one (by
 * index) is reported through first / first_got / first_want.
 * ------------------------------------------------------------------------ */
#include <pthread.h>

typedef struct {
  int op;
  orc_fmt f;
  int in_kind;
  const void *a, *b, *c;
  const void* got;
  size_t n, b0, b1; /* element count, block range [b0, b1) */
  uint64_t bad, first, first_got, first_want;
} orc_vjob;

static uint64_t in_enc(const orc_vjob* j, const void* p, size_t i) {
  if (j->in_kind == 0) return ((const uint32_t*)p)[i];
  return orc_encode((double)((const float*)p)[i], j->f.e, j->f.s, j->f.rn, j->f.ftz);
}

static void note_bad(orc_vjob* j, size_t i, uint64_t got, uint64_t want) {
  if (j->bad++ == 0 || i < j->first) {
    j->first = i;
    j->first_got = got;
    j->first_want = want;
  }
}

static void* orc_vthread(void* arg) {
  orc_vjob* j = (orc_vjob*)arg;
  const orc_fmt* f = &j->f;
  const unsigned nb = 1 + f->e + f->s;
  uint64_t want[1024];
  uint32_t blk[64 * 32];
  for (size_t b = j->b0; b < j->b1; ++b) {
    const size_t i0 = b * 1024;
    const size_t cnt = j->n - i0 < 1024 ? j->n - i0 : 1024;
    for (size_t k = 0; k < cnt; ++k) {
      const size_t i = i0 + k;
      const uint64_t x = in_enc(j, j->a, i);
      switch (j->op) {
        case 5: want[k] = x; break;
        case 6: {
          const float v = (float)orc_decode(x, f->e, f->s);
          uint32_t w;
          memcpy(&w, &v, 4);
          want[k] = w;
          break;
        }
        case ORC_MUL_ADD:
          want[k] = orc_mul_add(f->e, f->s, f->rn, f->ftz, x, in_enc(j, j->b, i), in_enc(j, j->c, i));
          break;
        default: want[k] = orc_binop(j->op, f->e, f->s, f->rn, f->ftz, x, in_enc(j, j->b, i)); break;
      }
    }
    if (j->op == 6) {
      const uint32_t* g = (const uint32_t*)j->got + i0;
      for (size_t k = 0; k < cnt; ++k)
        if (g[k] != (uint32_t)want[k]) note_bad(j, i0 + k, g[k], want[k]);
      continue;
    }
    for (size_t k = cnt; k < 1024; ++k) want[k] = 0; /* zero-filled tail, pack.hpp:50 */
    memset(blk, 0, nb * 128);
    for (unsigned k = 0; k < 1024; ++k)
      for (unsigned p = 0; p < nb; ++p) blk[p * 32 + (k >> 5)] |= (uint32_t)((want[k] >> p) & 1u) << (k & 31);
    const uint32_t* g = (const uint32_t*)j->got + b * nb * 32;
    if (memcmp(g, blk, nb * 128) != 0) {
      for (unsigned k = 0; k < cnt; ++k) {
        uint64_t v = 0;
        for (unsigned p = 0; p < nb; ++p) v |= (uint64_t)((g[p * 32 + (k >> 5)] >> (k & 31)) & 1u) << p;
        if (v != want[k]) note_bad(j, i0 + k, v, want[k]);
      }
    }
  }
  return NULL;
}

uint64_t orc_verify(int op, unsigned e, unsigned s, int rn, int ftz, int in_kind, const void* a,
                    const void* b, const void* c, const void* got, size_t n, int threads,
                    uint64_t* first, uint64_t* first_got, uint64_t* first_want) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  const size_t blocks = (n + 1023) / 1024;
  orc_vjob jobs[256];
  pthread_t tid[256];
  int started = 0;
  for (int t = 0; t < threads; ++t) {
    orc_vjob* j = &jobs[t];
    memset(j, 0, sizeof *j);
    j->op = op;
    j->f.e = e;
    j->f.s = s;
    j->f.rn = rn;
    j->f.ftz = ftz;
    j->in_kind = in_kind;
    j->a = a;
    j->b = b;
    j->c = c;
    j->got = got;
    j->n = n;
    j->b0 = blocks * (size_t)t / (size_t)threads;
    j->b1 = blocks * (size_t)(t + 1) / (size_t)threads;
    j->first = n;
    if (pthread_create(&tid[t], NULL, orc_vthread, j) == 0) {
      ++started;
    } else {
      orc_vthread(j); /* run inline */
      tid[t] = 0;
    }
  }
  uint64_t bad = 0, fi = n, fg = 0, fw = 0;
  for (int t = 0; t < threads; ++t) {
    if (tid[t]) pthread_join(tid[t], NULL);
    bad += jobs[t].bad;
    if (jobs[t].bad && jobs[t].first < fi) {
      fi = jobs[t].first;
      fg = jobs[t].first_got;
      fw = jobs[t].first_want;
    }
  }
  (void)started;
  if (first) *first = fi;
  if (first_got) *first_got = fg;
  if (first_want) *first_want = fw;
  return bad;
}

/* mul_add over ALL (a, b) pairs of a 16-bit format against nc fixed c values:
 * pair i of the chunk is a = a0 + i / 65536, b = i % 65536; result planes
 * got[k] hold bfp_add(bfp_mul(a, b), c_k) for the chunk's na * 65536 pairs.
 * The product is computed once per pair (orc_binop), each c through a
 * 65536-entry table add_tab[k * 65536 + p] = orc_binop(ADD, p, c_k). */
typedef struct {
  orc_fmt f;
  uint32_t a0;
  int nc;
  const uint16_t* add_tab;
  const uint32_t* const* got;
  size_t b0, b1;
  uint64_t bad, first, first_k, first_got, first_want;
} orc_pjob;

static void* orc_pthread(void* arg) {
  orc_pjob* j = (orc_pjob*)arg;
  const orc_fmt* f = &j->f;
  uint16_t prod[1024];
  for (size_t b = j->b0; b < j->b1; ++b) {
    for (unsigned k = 0; k < 1024; ++k) {
      const size_t i = b * 1024 + k;
      prod[k] = (uint16_t)orc_binop(ORC_MUL, f->e, f->s, f->rn, f->ftz, j->a0 + (i >> 16), i & 0xffff);
    }
    for (int q = 0; q < j->nc; ++q) {
      const uint16_t* tab = j->add_tab + (size_t)q * 65536;
      const uint32_t* g = j->got[q] + b * 16 * 32;
      for (unsigned w = 0; w < 32; ++w) {
        for (unsigned p = 0; p < 16; ++p) {
          uint32_t word = 0;
          for (unsigned t = 0; t < 32; ++t) word |= (uint32_t)((tab[prod[w * 32 + t]] >> p) & 1u) << t;
          if (word != g[p * 32 + w]) {
            for (unsigned t = 0; t < 32; ++t) {
              const unsigned k = w * 32 + t;
              uint64_t v = 0;
              for (unsigned pp = 0; pp < 16; ++pp) v |= (uint64_t)((g[pp * 32 + w] >> t) & 1u) << pp;
              const uint64_t want = tab[prod[k]];
              if (v != want && (j->bad++ == 0)) {
                j->first = b * 1024 + k;
                j->first_k = (uint64_t)q;
                j->first_got = v;
                j->first_want = want;
              }
            }
            break; /* this word's 32 elements are counted once */
          }
        }
      }
    }
  }
  return NULL;
}

uint64_t orc_verify_mul_add_pairs(unsigned e, unsigned s, int rn, int ftz, uint32_t a0, uint32_t na,
                                  const uint16_t* add_tab, int nc, const uint32_t* const* got, int threads,
                                  uint64_t* info /* first index, c slot, got, want */) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  const size_t blocks = (size_t)na * 64; /* na * 65536 pairs / 1024 */
  orc_pjob jobs[256];
  pthread_t tid[256];
  for (int t = 0; t < threads; ++t) {
    orc_pjob* j = &jobs[t];
    memset(j, 0, sizeof *j);
    j->f.e = e;
    j->f.s = s;
    j->f.rn = rn;
    j->f.ftz = ftz;
    j->a0 = a0;
    j->nc = nc;
    j->add_tab = add_tab;
    j->got = got;
    j->b0 = blocks * (size_t)t / (size_t)threads;
    j->b1 = blocks * (size_t)(t + 1) / (size_t)threads;
    if (pthread_create(&tid[t], NULL, orc_pthread, j) != 0) {
      orc_pthread(j);
      tid[t] = 0;
    }
  }
  uint64_t bad = 0;
  int have = 0;
  for (int t = 0; t < threads; ++t) {
    if (tid[t]) pthread_join(tid[t], NULL);
    if (jobs[t].bad && !have && info) {
      info[0] = jobs[t].first;
      info[1] = jobs[t].first_k;
      info[2] = jobs[t].first_got;
      info[3] = jobs[t].first_want;
      have = 1;
    }
    bad += jobs[t].bad;
  }
  return bad;
}

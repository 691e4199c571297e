// tests/native/ref_backend_test.cpp -- TEST: the reference-side binding
// (integration/bfp/gpu_backend.hpp) compiled against the UNMODIFIED reference
// headers, run on the GPU, byte-compared with the reference's own operators.
//
// For every compiled format x {RN, RZ} x {gradual, FTZ}: batches of
// bfp_vector<lane<1024>> operands built with field_from_elements
// (bitfield.hpp:33-43) from random + directed encodings, then
//   bfp_add / bfp_sub / bfp_mul / bfp_div (arith.hpp:235-444) and
//   bfp_add(bfp_mul(a, b), c)
// through the reference templates on the host and through the adapter
// (one vector per call and a batch per call) on the B200.  The resulting
// bitfields must be identical (bitfield operator==, every lane); error
// behaviour: mismatched specs throw std::invalid_argument like the reference.
//
// Built by oracle/Makefile (target `backend`) where /root/reference exists;
// the binary travels to the GPU box prebuilt (oracle/_ref/).
#include <bfp/gpu_backend.hpp>

#include <cstdio>
#include <random>

using namespace bfp;
using V = bfp_vector<lane<1024>>;

static std::vector<std::uint64_t> encodings(unsigned e, unsigned s, std::mt19937_64& rng) {
  const unsigned nb = 1 + e + s;
  const std::uint64_t mask = nb == 64 ? ~0ull : (1ull << nb) - 1;
  std::vector<std::uint64_t> v(1024);
  for (unsigned k = 0; k < 1024; ++k) {
    std::uint64_t x = rng() & mask;
    switch (k % 8) {  // weight the branch points: zero/subnormal, near overflow, specials
      case 0: x &= ~(((1ull << e) - 1) << s) | (std::uint64_t(rng() % 3) << s); break;
      case 1: x |= ((1ull << e) - 1 - rng() % 3) << s; break;
      case 2: x = (x & (1ull << (e + s))) | (((1ull << e) - 1) << s) | ((rng() & 1) << (s - 1)); break;
      default: break;
    }
    v[k] = x & mask;
  }
  v[0] = 0;
  v[1] = 1ull << (e + s);
  return v;
}

static V make(const format_spec& f, const std::vector<std::uint64_t>& enc) {
  return V{f, field_from_elements<lane<1024>>(f.total_bits(), enc)};
}

int main() {
  const unsigned fmts[][2] = {{3, 2}, {4, 3}, {5, 3}, {5, 7}, {5, 10}, {6, 9}, {8, 7}, {8, 15}, {8, 23}};
  std::mt19937_64 rng(0x160204716ull);
  long cases = 0;
  for (auto [e, s] : fmts)
    for (int rn = 0; rn < 2; ++rn)
      for (int ftz = 0; ftz < 2; ++ftz) {
        const format_spec f = make_spec(e, s, rn ? rounding_mode::rn : rounding_mode::rz,
                                        ftz ? subnormal_policy::ftz : subnormal_policy::gradual);
        constexpr int B = 6;  // vectors per batch
        std::vector<V> xs, ys, cs;
        for (int k = 0; k < B; ++k) {
          xs.push_back(make(f, encodings(e, s, rng)));
          ys.push_back(make(f, encodings(e, s, rng)));
          cs.push_back(make(f, encodings(e, s, rng)));
        }
        for (int op = 0; op < 5; ++op) {
          const auto got = gpu_backend::arith_batch(op, xs, ys, op == 4 ? &cs : nullptr);
          for (int k = 0; k < B; ++k) {
            V want;
            switch (op) {
              case 0: want = bfp_add(xs[k], ys[k]); break;
              case 1: want = bfp_sub(xs[k], ys[k]); break;
              case 2: want = bfp_mul(xs[k], ys[k]); break;
              case 3: want = bfp_div(xs[k], ys[k]); break;
              default: want = bfp_add(bfp_mul(xs[k], ys[k]), cs[k]); break;
            }
            V one;
            switch (op) {  // the one-vector-per-call entry points too
              case 0: one = bfp_add_gpu(xs[k], ys[k]); break;
              case 1: one = bfp_sub_gpu(xs[k], ys[k]); break;
              case 2: one = bfp_mul_gpu(xs[k], ys[k]); break;
              case 3: one = bfp_div_gpu(xs[k], ys[k]); break;
              default: one = bfp_mul_add_gpu(xs[k], ys[k], cs[k]); break;
            }
            if (!(got[k].field == want.field) || !(one.field == want.field) || !(got[k].spec == want.spec)) {
              for (unsigned i = 0; i < 1024; ++i) {
                const auto a = element_of(got[k].field, i), b = element_of(want.field, i);
                if (a != b) {
                  std::printf("FAIL 1/%u/%u rn=%d ftz=%d op=%d vec=%d elem=%u: x=%#llx y=%#llx gpu=%#llx ref=%#llx\n",
                              e, s, rn, ftz, op, k, i, (unsigned long long)element_of(xs[k].field, i),
                              (unsigned long long)element_of(ys[k].field, i), (unsigned long long)a,
                              (unsigned long long)b);
                  return 1;
                }
              }
              std::printf("FAIL 1/%u/%u op=%d: single-call result differs\n", e, s, op);
              return 1;
            }
            ++cases;
          }
        }
      }
  // reference error behaviour: specs differing only in the name are rejected
  const format_spec a = make_spec(4, 3), b = make_spec(4, 3, rounding_mode::rn, subnormal_policy::gradual, "other");
  const V x = make(a, encodings(4, 3, rng)), y = make(b, encodings(4, 3, rng));
  bool threw = false;
  try {
    (void)bfp_mul_gpu(x, y);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  if (!threw) {
    std::printf("FAIL: mismatched specs accepted\n");
    return 1;
  }
  std::printf("ok %ld vector results (1024 elements each) identical to the reference\n", cases);
  return 0;
}

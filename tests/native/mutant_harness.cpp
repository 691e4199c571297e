// tests/native/mutant_harness.cpp -- TEST HARNESS ONLY (tests/test_mutation.py).
// The RN + gradual networks of one format (-DMUT_E, -DMUT_S, -DMUT_GEN =
// "gen/gen_E_S.cuh") -- the templates of bfp_circuits.cuh (ops 0..4) and
// their generated LOP3 covers (ops 10..14; 15 = mul_add's fast-domain
// cover inside its domain, the general cover outside) -- compiled for the host from a
// directory given by -I, so a test can compile a deliberately corrupted copy
// (one flipped LUT bit, a broken rounding rule) and show that the parity
// checks catch it.
#include <cstddef>
#include <cstdint>

#include "bfp_circuits.cuh"
#include MUT_GEN

using namespace bfpg;
using F = Format<MUT_E, MUT_S, true, false>;

extern "C" int mut_binop(int op, const uint32_t* x, const uint32_t* y, const uint32_t* c, uint32_t* z,
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
        case 0: add_w<F, false>(X, Y, Z); break;
        case 1: add_w<F, true>(X, Y, Z); break;
        case 2: mul_w<F>(X, Y, Z); break;
        case 3: div_w<F>(X, Y, Z); break;
        case 4: mul_add_w<F>(X, Y, C, Z); break;
        case 10: Gen<F, 0>::run(X, Y, C, Z); break;
        case 11: Gen<F, 1>::run(X, Y, C, Z); break;
        case 12: Gen<F, 2>::run(X, Y, C, Z); break;
        case 13: Gen<F, 3>::run(X, Y, C, Z); break;
        case 14: Gen<F, 4>::run(X, Y, C, Z); break;
        case 15: {  // mul_add as the kernels run it, lane by lane: the fast-domain cover
                    // wherever the predicate allows it, the general cover elsewhere
          if constexpr (Gen<F, 5>::ok) {
            w32 G[N];
            Gen<F, 4>::run(X, Y, C, G);
            Gen<F, 5>::run(X, Y, C, Z);
            const w32 dom = mul_add_fast_domain<F>(X, Y, C);
            for (int j = 0; j < N; ++j) Z[j] = (Z[j] & dom) | (G[j] & ~dom);
          } else {
            return 1;
          }
          break;
        }
        default: return 1;
      }
      for (int j = 0; j < N; ++j) z[(b * N + j) * 32 + t] = Z[j];
    }
  return 0;
}

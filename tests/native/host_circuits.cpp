// tests/native/host_circuits.cpp -- TEST HARNESS ONLY.
// Compiles the device networks (paper_1602_04716_b200/csrc/bfp_circuits.cuh)
// for the host so tests can check them exhaustively against the oracle on a
// machine without a GPU.  Operands use the device plane layout.
#include <cstddef>
#include <cstdint>

#include "../../paper_1602_04716_b200/csrc/bfp_circuits.cuh"
#include "../../paper_1602_04716_b200/csrc/bfp_formats.h"

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
        case 0: add_w<F, false>(X, Y, Z); break;
        case 1: add_w<F, true>(X, Y, Z); break;
        case 2: mul_w<F>(X, Y, Z); break;
        case 4: mul_add_w<F>(X, Y, C, Z); break;
        default: return;
      }
      for (int j = 0; j < N; ++j) z[(b * N + j) * 32 + t] = Z[j];
    }
}

extern "C" int host_binop(int op, unsigned e, unsigned s, int rn, int ftz, const uint32_t* x,
                          const uint32_t* y, const uint32_t* c, uint32_t* z, size_t nblocks) {
#define DISPATCH(E_, S_)                                                          \
  if (e == E_ && s == S_) {                                                       \
    if (rn && !ftz) run<Format<E_, S_, true, false>>(op, x, y, c, z, nblocks);    \
    if (rn && ftz) run<Format<E_, S_, true, true>>(op, x, y, c, z, nblocks);      \
    if (!rn && !ftz) run<Format<E_, S_, false, false>>(op, x, y, c, z, nblocks);  \
    if (!rn && ftz) run<Format<E_, S_, false, true>>(op, x, y, c, z, nblocks);    \
    return 0;                                                                     \
  }
  BFP_FORMAT_LIST(DISPATCH)
#undef DISPATCH
  return 4;
}

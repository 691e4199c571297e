// Random-operand check of the TEMPLATE networks (the ones NVRTC compiles for
// runtime formats) over a grid of formats, including narrow-exponent /
// wide-significand ones whose working exponent needs more than E + 2 bits,
// against the oracle (liboracle.so).  Built and run by
// tests/test_circuits_host.py::test_template_format_sweep; prints "total bad N".
#include "../../paper_1602_04716_b200/csrc/bfp_circuits.cuh"
#include <cstdio>
#include <random>
extern "C" uint64_t orc_binop(int op, unsigned e, unsigned s, int rn, int ftz, uint64_t x, uint64_t y);
using namespace bfpg;
long total_bad = 0;
template <class F> void run() {
  constexpr int N = F::N;
  std::mt19937_64 r(F::E * 100 + F::S);
  long bad[4] = {0, 0, 0, 0};
  for (int it = 0; it < 3000; ++it) {
    uint64_t xs[32], ys[32];
    w32 X[N] = {}, Y[N] = {};
    for (int k = 0; k < 32; ++k) {
      xs[k] = r() & ((1ull << N) - 1); ys[k] = r() & ((1ull << N) - 1);
      if (k & 1) xs[k] &= ~(((1ull << F::E) - 1) << F::S) | (uint64_t(r() & 1) << F::S);  // subnormal-ish
      if (k & 2) ys[k] &= ~(((1ull << F::E) - 1) << F::S) | (uint64_t(r() & 1) << F::S);
      for (int j = 0; j < N; ++j) { X[j] |= w32((xs[k] >> j) & 1) << k; Y[j] |= w32((ys[k] >> j) & 1) << k; }
    }
    for (int op = 0; op < 4; ++op) {
      w32 Z[N];
      if (op == 0) add_w<F, false>(X, Y, Z); else if (op == 1) add_w<F, true>(X, Y, Z);
      else if (op == 2) mul_w<F>(X, Y, Z); else div_w<F>(X, Y, Z);
      for (int k = 0; k < 32; ++k) {
        uint64_t z = 0; for (int j = 0; j < N; ++j) z |= uint64_t((Z[j] >> k) & 1) << j;
        if (z != orc_binop(op, F::E, F::S, F::RN, F::FTZ, xs[k], ys[k])) ++bad[op];
      }
    }
  }
  const long b = bad[0] + bad[1] + bad[2] + bad[3];
  total_bad += b;
  if (b) printf("1/%d/%d rn=%d ftz=%d: add %ld sub %ld mul %ld div %ld\n", F::E, F::S, F::RN, F::FTZ, bad[0], bad[1], bad[2], bad[3]);
}
template <int E, int S> void fmt() { run<Format<E, S, true, false>>(); run<Format<E, S, false, true>>(); }
template <int E, int... Ss> void row() { (fmt<E, Ss>(), ...); }
int main() {
  row<2, 1, 2, 3, 5, 8, 11, 16, 23, 24>();
  row<3, 1, 2, 4, 7, 11, 16, 20, 24>();
  row<4, 1, 3, 6, 12, 18, 24>();
  row<5, 2, 10, 17, 24>();
  row<6, 1, 9, 24>();
  row<7, 3, 20, 24>();
  row<8, 1, 7, 23>();
  row<9, 5, 20>();
  row<10, 1, 24>();
  row<11, 4, 24>();
  printf("total bad %ld\n", total_bad);
}

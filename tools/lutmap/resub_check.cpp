// tools/lutmap/resub_check.cpp -- exhaustive check of the post-mapping optimiser
// (resub.hpp) on the small formats: every input combination of the optimised
// LUT network against the AND/XOR graph of the template it came from.
//   g++ -O2 -std=c++17 -Itools/lutmap -Ipaper_1602_04716_b200/csrc tools/lutmap/resub_check.cpp -o resub_check
// Prints one line per network: "<name> mapped <a> optimised <b> patterns <n> ok|MISMATCH"; exit 1 on a mismatch.
#include "resub.hpp"
#define BFP_SYMBOLIC_WORD lutmap::Sym
#include "bfp_circuits.cuh"

#include <cstdio>

using namespace bfpg;

static int failures = 0;

template <class F>
void check(int op, const char* name) {
  lutmap::Graph g;
  lutmap::graph() = &g;
  constexpr int N = F::N;
  const int nops = op == 4 ? 3 : 2;
  w32 X[N], Y[N], Cc[N], Z[N];
  for (int i = 0; i < N; ++i) X[i] = lutmap::Sym::of(g.input());
  for (int i = 0; i < N; ++i) Y[i] = lutmap::Sym::of(g.input());
  for (int i = 0; i < N; ++i) Cc[i] = op == 4 ? lutmap::Sym::of(g.input()) : lutmap::Sym(0u);
  switch (op) {
    case 0: add_w<F, false>(X, Y, Z); break;
    case 1: add_w<F, true>(X, Y, Z); break;
    case 2: mul_w<F>(X, Y, Z); break;
    case 3: div_w<F>(X, Y, Z); break;
    default: mul_add_w<F>(X, Y, Cc, Z); break;
  }
  std::vector<lutmap::Lit> outs;
  for (int i = 0; i < N; ++i) outs.push_back(Z[i].l);
  auto M = lutmap::map_luts(g, outs);
  lutmap::recover_area(g, M, outs);
  lutmap::LutNet net = lutmap::from_mapping(g, M, outs);
  const size_t mapped = lutmap::count_luts(net);
  lutmap::optimize_net(net);
  const size_t optimised = lutmap::count_luts(net);
  const int bits = nops * N;
  const uint64_t patterns = 1ull << bits;
  const int rounds = int(patterns >> 6) > 0 ? int(patterns >> 6) : 1;
  const bool ok = lutmap::equivalent_on(g, outs, net, rounds, [&](int r, std::vector<uint64_t>& pis) {
    for (int j = 0; j < bits; ++j) {
      uint64_t w = 0;
      for (int b = 0; b < 64; ++b)
        if ((((uint64_t(r) << 6) | uint64_t(b)) >> j) & 1) w |= 1ull << b;
      pis[size_t(j)] = w;
    }
  });
  std::printf("%s mapped %zu optimised %zu patterns %llu %s\n", name, mapped, optimised,
              (unsigned long long)patterns, ok ? "ok" : "MISMATCH");
  if (!ok || optimised > mapped) ++failures;
  lutmap::graph() = nullptr;
}

int main() {
  check<Format<3, 2, true, false>>(0, "1/3/2 add rn");
  check<Format<3, 2, true, false>>(1, "1/3/2 sub rn");
  check<Format<3, 2, true, false>>(2, "1/3/2 mul rn");
  check<Format<3, 2, true, false>>(3, "1/3/2 div rn");
  check<Format<3, 2, false, true>>(4, "1/3/2 mul_add rz ftz");
  check<Format<4, 3, true, false>>(0, "1/4/3 add rn");
  check<Format<4, 3, false, true>>(1, "1/4/3 sub rz ftz");
  check<Format<4, 3, true, false>>(2, "1/4/3 mul rn");
  check<Format<4, 3, true, true>>(3, "1/4/3 div rn ftz");
  check<Format<4, 3, true, false>>(4, "1/4/3 mul_add rn");
  return failures ? 1 : 0;
}

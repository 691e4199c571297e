// tools/lutmap/count.cpp -- LOP3 count of the mapped networks, per format x op.
//   g++ -O2 -std=c++17 -I... count.cpp && ./a.out
#include "resub.hpp"
#define BFP_SYMBOLIC_WORD lutmap::Sym
#include "bfp_circuits.cuh"

#include <cstdio>

using namespace bfpg;

template <class F>
size_t count(int op, size_t* gates) {
  lutmap::Graph g;
  lutmap::graph() = &g;
  constexpr int N = F::N;
  w32 X[N], Y[N], Cc[N], Z[N];
  for (int i = 0; i < N; ++i) X[i] = lutmap::Sym::of(g.input());
  for (int i = 0; i < N; ++i) Y[i] = lutmap::Sym::of(g.input());
  for (int i = 0; i < N; ++i) Cc[i] = lutmap::Sym::of(g.input());
  switch (op) {
    case 0: add_w<F, false>(X, Y, Z); break;
    case 1: add_w<F, true>(X, Y, Z); break;
    case 2: mul_w<F>(X, Y, Z); break;
    case 3: div_w<F>(X, Y, Z); break;
    default: mul_add_w<F>(X, Y, Cc, Z); break;
  }
  std::vector<lutmap::Lit> outs;
  for (int i = 0; i < N; ++i) outs.push_back(Z[i].l);
  const lutmap::LutNet net = lutmap::optimised_cover(g, outs);
  *gates = g.nodes.size();
  lutmap::graph() = nullptr;
  return lutmap::count_luts(net);
}

template <int E, int S>
void row() {
  for (int op = 0; op < 5; ++op) {
    size_t gates;
    const size_t l = count<Format<E, S, true, false>>(op, &gates);
    std::printf("1/%d/%d op%d: mapped LOP3 %zu (%.2f/elem), AIG nodes %zu\n", E, S, op, l, l / 32.0, gates);
  }
}

int main() {
  row<3, 2>();
  row<4, 3>();
  row<5, 10>();
  row<8, 15>();
  return 0;
}

// tools/lutmap/stages.cpp -- LUTs of the mapped networks per circuit stage
// (BFP_STAGE markers in bfp_circuits.cuh): where the LOP3s of a kernel go.
//   g++ -O2 -std=c++17 -Itools/lutmap -Ipaper_1602_04716_b200/csrc tools/lutmap/stages.cpp -o /tmp/stages
//   /tmp/stages
#include "lutmap.hpp"
#define BFP_SYMBOLIC_WORD lutmap::Sym
#define BFP_STAGE(name) lutmap::graph()->stage(name)
#include "bfp_circuits.cuh"

#include <cstdio>
#include <map>

using namespace bfpg;

template <class F>
void report(int op, const char* title) {
  lutmap::Graph g;
  lutmap::graph() = &g;
  constexpr int N = F::N;
  w32 X[N], Y[N], Cc[N], Z[N];
  for (int i = 0; i < N; ++i) X[i] = lutmap::Sym::of(g.input());
  for (int i = 0; i < N; ++i) Y[i] = lutmap::Sym::of(g.input());
  for (int i = 0; i < N; ++i) Cc[i] = lutmap::Sym::of(g.input());
  g.stage("(entry)");
  switch (op) {
    case 0: add_w<F, false>(X, Y, Z); break;
    case 2: mul_w<F>(X, Y, Z); break;
    case 3: div_w<F>(X, Y, Z); break;
    default: mul_add_w<F>(X, Y, Cc, Z); break;
  }
  std::vector<lutmap::Lit> outs;
  for (int i = 0; i < N; ++i) outs.push_back(Z[i].l);
  auto M = lutmap::map_luts(g, outs);
  lutmap::recover_area(g, M, outs);
  std::map<std::string, int> per;
  for (uint32_t v : M.required) per[g.stage_names[g.tag[v]]]++;
  std::printf("%s: %zu LUTs\n", title, M.luts);
  for (auto& [k, n] : per) std::printf("  %-28s %5d\n", k.c_str(), n);
  lutmap::graph() = nullptr;
}

int main() {
  report<Format<6, 9, true, false>>(4, "1/6/9 mul_add RN");
  report<Format<8, 15, true, false>>(2, "1/8/15 mul RN");
  report<Format<5, 10, true, false>>(2, "1/5/10 mul RN");
  report<Format<6, 9, true, false>>(0, "1/6/9 add RN");
  return 0;
}

// tools/lutmap/stages.cpp -- LUTs of the mapped networks per circuit stage, before / after resub.hpp
// (BFP_STAGE markers in bfp_circuits.cuh): where the LOP3s of a kernel go.
//   g++ -O2 -std=c++17 -Itools/lutmap -Ipaper_1602_04716_b200/csrc tools/lutmap/stages.cpp -o /tmp/stages
//   /tmp/stages
#include "resub.hpp"
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
  // structural cover (mapper alone) next to the shipped cover (after resub.hpp)
  const lutmap::LutNet plain = lutmap::optimised_cover(g, outs, false);
  const lutmap::LutNet opt = lutmap::optimised_cover(g, outs, true);
  std::map<std::string, std::pair<int, int>> per;
  for (uint32_t v : lutmap::live_order(plain)) per[g.stage_names[plain.nodes[v].tag]].first++;
  for (uint32_t v : lutmap::live_order(opt)) per[g.stage_names[opt.nodes[v].tag]].second++;
  std::printf("%s: %zu LUTs mapped, %zu after the post-mapping optimiser\n", title, lutmap::count_luts(plain),
              lutmap::count_luts(opt));
  for (auto& [k, n] : per) std::printf("  %-28s %5d %5d\n", k.c_str(), n.first, n.second);
  lutmap::graph() = nullptr;
}

int main() {
  report<Format<6, 9, true, false>>(4, "1/6/9 mul_add RN");
  report<Format<8, 15, true, false>>(2, "1/8/15 mul RN");
  report<Format<5, 10, true, false>>(2, "1/5/10 mul RN");
  report<Format<6, 9, true, false>>(0, "1/6/9 add RN");
  return 0;
}

// tools/lutmap/resub_try.cpp -- mapped LOP3 counts before / after the resubstitution pass.
//   g++ -O2 -std=c++17 -Itools/lutmap -Ipaper_1602_04716_b200/csrc tools/lutmap/resub_try.cpp -o /tmp/resub_try
#include "resub.hpp"
#define BFP_SYMBOLIC_WORD lutmap::Sym
#define BFP_STAGE(name) lutmap::graph()->stage(name)
#include "bfp_circuits.cuh"

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>

using namespace bfpg;
static bool g_odc = true;
static int g_iters = 0;
static int g_elim = 0;

template <class F>
void report(int op, const char* title, int passes, bool dc, bool two) {
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
  lutmap::LutNet net = lutmap::from_mapping(g, M, outs);
  const auto t0 = std::chrono::steady_clock::now();
  lutmap::Resub rs(net);
  const auto st = rs.run(passes, dc, two, g_odc);
  if (g_elim) {
    for (int it = 0; it < 4; ++it) {
      const int rem = lutmap::Resub(net).eliminate(dc, g_odc);
      const auto st3 = lutmap::Resub(net).run(passes, dc, two, g_odc);
      std::printf("  eliminate %d: removed %d, then resub -> %zu\n", it, rem, st3.after);
      if (rem == 0) break;
    }
  }
  size_t best = lutmap::count_luts(net);
  for (int it = 0; it < g_iters; ++it) {
    lutmap::Graph g2;
    g2.stage_names = g.stage_names;
    std::vector<lutmap::Lit> o2 = lutmap::to_graph(net, g2);
    auto M2 = lutmap::map_luts(g2, o2);
    lutmap::recover_area(g2, M2, o2);
    lutmap::LutNet n2 = lutmap::from_mapping(g2, M2, o2);
    const size_t remapped = lutmap::count_luts(n2);
    lutmap::Resub rs2(n2);
    const auto st2 = rs2.run(passes, dc, two, g_odc);
    std::printf("  iter %d: remap %zu -> resub %zu\n", it, remapped, st2.after);
    if (st2.after < best) {
      best = st2.after;
      net = n2;
    } else {
      break;
    }
  }
  const double sec = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  const bool ok = lutmap::equivalent_on_random(g, outs, net, 2000, 12345);
  std::printf("%s: mapped %zu -> %zu -> %zu LUTs (wires %d, one %d, two %d) %.1f s, random check %s\n", title, st.before,
              st.after, lutmap::count_luts(net), st.wires, st.one, st.two, sec, ok ? "ok" : "MISMATCH");
  std::map<std::string, int> per;
  for (uint32_t v : lutmap::live_order(net)) per[g.stage_names[net.nodes[v].tag]]++;
  for (auto& [k, n] : per) std::printf("  %-28s %5d\n", k.c_str(), n);
  lutmap::graph() = nullptr;
}

int main(int argc, char** argv) {
  const int passes = argc > 1 ? std::atoi(argv[1]) : 3;
  const bool dc = argc > 2 ? std::atoi(argv[2]) : true;
  const bool two = argc > 3 ? std::atoi(argv[3]) : true;
  g_odc = argc > 4 ? std::atoi(argv[4]) : true;
  g_iters = argc > 5 ? std::atoi(argv[5]) : 0;
  g_elim = argc > 6 ? std::atoi(argv[6]) : 0;
  report<Format<4, 3, true, false>>(4, "1/4/3 mul_add RN", passes, dc, two);
  report<Format<6, 9, true, false>>(0, "1/6/9 add RN", passes, dc, two);
  report<Format<6, 9, true, false>>(4, "1/6/9 mul_add RN", passes, dc, two);
  report<Format<8, 15, true, false>>(2, "1/8/15 mul RN", passes, dc, two);
  return 0;
}

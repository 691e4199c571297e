// tools/lutmap/resub.hpp -- post-mapping optimisation of a LOP3 cover.
//
// The structural mapper (lutmap.hpp) can only place LUT boundaries on nodes of
// the AND/XOR graph it was given.  This pass works on the mapped network
// itself: for every LUT r it builds a window (a cut of at most CUT signals
// below r, every node computable from that cut, exact truth tables over the
// cut), and tries to re-express r's function with fewer LUTs than the cone r
// alone keeps alive (its maximum fanout-free cone):
//   * as an existing signal or its complement (the cone disappears),
//   * as ONE LUT over any three signals of the window (Boolean
//     resubstitution: the inputs need not be the cone's own leaves),
//   * as TWO LUTs g(h(a,b,c), d, e) when the cone holds three or more.
// Input combinations of the window cut that cannot occur (satisfiability
// don't-cares) are found exactly by enumerating a second, deeper cut: treating
// that cut's signals as free variables over-approximates what can reach the
// window, so every replacement is sound by construction.  Every accepted move
// is a function-preserving rewrite on all reachable inputs; gen.cpp
// additionally cross-checks the final network against the AND/XOR graph on
// random words, and the test suite checks the emitted covers like any network.
#pragma once

#include "lutmap.hpp"

#include <cstring>
#include <random>

namespace lutmap {

struct LNode {
  uint8_t n = 0;  // fanins (0 for const / PI)
  uint32_t in[3] = {0, 0, 0};
  uint8_t tt = 0;  // over (in[0], in[1], in[2]) = lop3 (a, b, c)
  uint16_t tag = 0;
  double ord = 0;  // position in the template's own evaluation order (emission order key)
};

struct LutNet {
  uint32_t n_pi = 0;
  std::vector<LNode> nodes;   // 0 = const 0, 1..n_pi = inputs, then LUTs (any order; acyclic)
  std::vector<uint32_t> outs; // literal = id * 2 + complement
  bool is_lut(uint32_t v) const { return v > n_pi; }
};

// value of an 8-bit lop3 table on three words
template <class W>
inline W lut_eval(uint8_t tt, W a, W b, W c) {
  W r = W(0);
  for (int k = 0; k < 8; ++k)
    if ((tt >> k) & 1) r |= ((k & 4) ? a : ~a) & ((k & 2) ? b : ~b) & ((k & 1) ? c : ~c);
  return r;
}

inline LutNet from_mapping(const Graph& g, const Mapping& M, const std::vector<Lit>& outputs) {
  LutNet net;
  std::vector<uint32_t> id(g.nodes.size(), 0);
  net.nodes.push_back(LNode{});
  for (size_t v = 1; v < g.nodes.size(); ++v)
    if (g.nodes[v].kind == 1) {
      net.nodes.push_back(LNode{});
      id[v] = uint32_t(net.nodes.size() - 1);
    }
  net.n_pi = uint32_t(net.nodes.size() - 1);
  for (uint32_t v : M.required) {  // ascending graph ids = topological
    const Cut& c = M.cuts[v][M.best[v]];
    LNode l;
    l.n = c.n;
    for (int k = 0; k < c.n; ++k) l.in[k] = id[c.leaf[k]];
    l.tt = c.tt;
    l.tag = g.tag[v];
    l.ord = double(v);
    net.nodes.push_back(l);
    id[v] = uint32_t(net.nodes.size() - 1);
  }
  for (Lit o : outputs) net.outs.push_back(id[o >> 1] * 2 + (o & 1));
  return net;
}

// Topological order of the live LUTs (reachable from the outputs).
inline std::vector<uint32_t> live_order(const LutNet& net) {
  std::vector<uint32_t> order;
  std::vector<char> st(net.nodes.size(), 0);
  std::vector<std::pair<uint32_t, int>> stack;
  for (uint32_t o : net.outs) {
    if (!net.is_lut(o >> 1) || st[o >> 1]) continue;
    stack.push_back({o >> 1, 0});
    st[o >> 1] = 1;
    while (!stack.empty()) {
      auto& [v, k] = stack.back();
      if (k < net.nodes[v].n) {
        const uint32_t u = net.nodes[v].in[k++];
        if (net.is_lut(u) && !st[u]) {
          st[u] = 1;
          stack.push_back({u, 0});
        }
      } else {
        order.push_back(v);
        stack.pop_back();
      }
    }
  }
  return order;
}

inline size_t count_luts(const LutNet& net) { return live_order(net).size(); }

// The live LUTs in the template's own evaluation order as far as the
// dependencies allow (smallest `ord` first among the ready nodes): the order
// the straight-line code is emitted in.  (A depth-first order from the outputs
// lengthens live ranges; ptxas starts from the source order.)
inline std::vector<uint32_t> natural_order(const LutNet& net) {
  const std::vector<uint32_t> live = live_order(net);
  std::vector<int> pending(net.nodes.size(), -1);
  std::vector<std::vector<uint32_t>> users(net.nodes.size());
  for (uint32_t v : live) {
    int p = 0;
    const LNode& l = net.nodes[v];
    for (int k = 0; k < l.n; ++k) {
      bool dup = false;
      for (int j = 0; j < k; ++j) dup |= l.in[j] == l.in[k];
      if (!dup && net.is_lut(l.in[k])) {
        ++p;
        users[l.in[k]].push_back(v);
      }
    }
    pending[v] = p;
  }
  auto later = [&](uint32_t a, uint32_t b) {
    return net.nodes[a].ord != net.nodes[b].ord ? net.nodes[a].ord > net.nodes[b].ord : a > b;
  };
  std::vector<uint32_t> heap;
  for (uint32_t v : live)
    if (pending[v] == 0) heap.push_back(v);
  std::make_heap(heap.begin(), heap.end(), later);
  std::vector<uint32_t> order;
  while (!heap.empty()) {
    std::pop_heap(heap.begin(), heap.end(), later);
    const uint32_t v = heap.back();
    heap.pop_back();
    order.push_back(v);
    for (uint32_t u : users[v])
      if (--pending[u] == 0) {
        heap.push_back(u);
        std::push_heap(heap.begin(), heap.end(), later);
      }
  }
  return order;
}

// Net vs graph on 64 patterns per round; fill(round, words) sets one word per
// primary input (bit b of every word = pattern b).
template <class Fill>
inline bool equivalent_on(const Graph& g, const std::vector<Lit>& outputs, const LutNet& net, int rounds,
                          Fill fill) {
  const auto order = live_order(net);
  std::vector<uint64_t> pis(net.n_pi);
  for (int r = 0; r < rounds; ++r) {
    fill(r, pis);
    std::vector<uint64_t> gv(g.nodes.size(), 0), nv(net.nodes.size(), 0);
    uint32_t pi = 0;
    for (size_t v = 1; v < g.nodes.size(); ++v) {
      const Node& nd = g.nodes[v];
      if (nd.kind == 1) {
        gv[v] = pis[pi];
        nv[++pi] = gv[v];
      } else if (nd.kind >= 2) {
        const uint64_t a = gv[nd.a >> 1] ^ ((nd.a & 1) ? ~0ull : 0ull);
        const uint64_t b = gv[nd.b >> 1] ^ ((nd.b & 1) ? ~0ull : 0ull);
        gv[v] = nd.kind == 2 ? (a & b) : (a ^ b);
      }
    }
    for (uint32_t v : order) {
      const LNode& l = net.nodes[v];
      nv[v] = lut_eval<uint64_t>(l.tt, l.n > 0 ? nv[l.in[0]] : 0, l.n > 1 ? nv[l.in[1]] : 0,
                                 l.n > 2 ? nv[l.in[2]] : 0);
    }
    for (size_t i = 0; i < outputs.size(); ++i) {
      const uint64_t a = gv[outputs[i] >> 1] ^ ((outputs[i] & 1) ? ~0ull : 0ull);
      const uint64_t b = nv[net.outs[i] >> 1] ^ ((net.outs[i] & 1) ? ~0ull : 0ull);
      if (a != b) return false;
    }
  }
  return true;
}

// Independent random words per input: a mix of uniform and sparse / dense
// words so that all-ones and all-zero fields show up.
inline bool equivalent_on_random(const Graph& g, const std::vector<Lit>& outputs, const LutNet& net,
                                 int rounds, uint64_t seed) {
  std::mt19937_64 rng(seed);
  return equivalent_on(g, outputs, net, rounds, [&](int, std::vector<uint64_t>& pis) {
    for (uint64_t& w : pis) {
      w = rng();
      const int mode = int(rng() % 4);
      if (mode == 1) w &= rng() & rng();
      if (mode == 2) w |= rng() | rng();
    }
  });
}

// Operands drawn as floating-point encodings of `nops` operands of n = 1 + e + s
// planes each (plane order: fraction LSB first, exponent, sign): exponent and
// fraction classes weighted towards the special and boundary values, and
// operands correlated with each other (equal, negated, adjacent exponents) so
// that cancellation, ties and the subnormal range are exercised.
inline bool equivalent_on_operands(const Graph& g, const std::vector<Lit>& outputs, const LutNet& net,
                                   int rounds, uint64_t seed, int e, int s, int nops) {
  std::mt19937_64 rng(seed);
  const int n = 1 + e + s;
  const uint64_t emax = (1ull << e) - 1, fmax = (1ull << s) - 1;
  auto field = [&](uint64_t top) -> uint64_t {
    switch (rng() % 8) {
      case 0: return 0;
      case 1: return top;
      case 2: return 1;
      case 3: return top - 1;
      case 4: return top >> 1;
      case 5: return (top >> 1) + 1;
      default: return rng() & top;
    }
  };
  return equivalent_on(g, outputs, net, rounds, [&](int, std::vector<uint64_t>& pis) {
    for (uint64_t& w : pis) w = 0;
    for (int lane = 0; lane < 64; ++lane) {
      uint64_t enc[3] = {0, 0, 0};
      for (int k = 0; k < nops; ++k) {
        uint64_t ex = field(emax), fr = field(fmax), sg = rng() & 1;
        if (k > 0) {
          const uint64_t pe = (enc[k - 1] >> s) & emax, pf = enc[k - 1] & fmax;
          switch (rng() % 8) {
            case 0: ex = pe; fr = pf; break;                              // equal magnitude
            case 1: ex = pe; break;                                        // same exponent
            case 2: ex = pe < emax ? pe + 1 : pe; break;                   // adjacent exponents
            case 3: ex = pe > 0 ? pe - 1 : pe; break;
            case 4: ex = (emax - 1) - (pe < emax ? pe : emax - 1); break;  // product near 1 / near the range ends
            case 5: ex = pe; fr = pf ^ 1; break;
            default: break;
          }
        }
        enc[k] = (sg << (e + s)) | (ex << s) | fr;
      }
      for (int k = 0; k < nops; ++k)
        for (int j = 0; j < n; ++j)
          if ((enc[k] >> j) & 1) pis[size_t(k) * n + j] |= 1ull << lane;
    }
  });
}

struct ResubStats {
  int wires = 0, one = 0, two = 0, merged = 0;
  size_t before = 0, after = 0;
};

class Resub {
 public:
#ifndef RESUB_CUT
#define RESUB_CUT 10
#endif
#ifndef RESUB_DEEP
#define RESUB_DEEP 16
#endif
  static constexpr int CUT = RESUB_CUT;    // window cut size
  static constexpr int WORDS = (1 << CUT) / 64;
  static constexpr int DEEP = RESUB_DEEP;  // deeper cut for the care set
  using TT = std::array<uint64_t, WORDS>;

  explicit Resub(LutNet& n) : net(n) {}

#ifndef RESUB_ODC_DEPTH
#define RESUB_ODC_DEPTH 2
#endif
  static constexpr int ODC_DEPTH = RESUB_ODC_DEPTH;
#ifndef RESUB_D1
#define RESUB_D1 64
#endif
#ifndef RESUB_D2
#define RESUB_D2 24
#endif
#ifndef RESUB_D3
#define RESUB_D3 32
#endif
#ifndef RESUB_ELIM_MIN_GAIN
#define RESUB_ELIM_MIN_GAIN 0
#endif
  static constexpr int ELIM_MIN_GAIN = RESUB_ELIM_MIN_GAIN;
  bool use_odc_ = true;
  ResubStats run(int passes = 3, bool use_dc = true, bool two_lut = true, bool use_odc = true) {
    ResubStats st;
    use_odc_ = use_odc;
    st.before = count_luts(net);
    for (int p = 0; p < passes; ++p) {
      bool any = false;
      analyse();
      std::vector<uint32_t> roots = order_;
      for (uint32_t r : roots) {
        if (refs_[r] == 0) continue;  // removed by an earlier move of this pass
        if (try_root(r, use_dc, two_lut, st)) {
          any = true;
          analyse();
        }
      }
      if (!any) break;
    }
    st.after = count_luts(net);
    return st;
  }

  // Node elimination: a LUT t with two or three users and a fanout-free cone
  // of one cannot be removed by re-expressing any single root.  Here every
  // user of t is re-expressed over window signals other than t (one LUT each,
  // never growing the network); when all succeed t and whatever only it kept
  // alive disappear.  Returns the number of LUTs removed.
  int eliminate(bool use_dc = true, bool use_odc = true) {
    use_odc_ = use_odc;
    analyse();
    int removed = 0;
    ResubStats scratch;
    const std::vector<uint32_t> nodes = order_;
    for (uint32_t t : nodes) {
      if (refs_[t] == 0 || is_po_[t]) continue;
      const std::vector<uint32_t> users = fanouts_[t];
      if (users.size() < 2 || users.size() > 5) continue;
      const size_t before = order_.size();
      const LutNet backup = net;
      forbid_ = t;
      min_gain_ = ELIM_MIN_GAIN;
      bool ok = true;
      for (uint32_t u : users) {
        if (refs_[u] == 0) continue;
        bool uses_t = false;
        for (int j = 0; j < net.nodes[u].n; ++j) uses_t |= net.nodes[u].in[j] == t;
        if (!uses_t) continue;
        if (!try_root(u, use_dc, true, scratch)) {
          ok = false;
          break;
        }
        analyse();
      }
      forbid_ = 0;
      min_gain_ = 1;
      if (ok) {
        analyse();
        if (order_.size() < before) {
          removed += int(before - order_.size());
          continue;
        }
      }
      net = backup;
      analyse();
    }
    return removed;
  }

 private:
  LutNet& net;
  uint32_t forbid_ = 0;  // eliminate(): the node the new expression must not use
  int min_gain_ = 1;
  std::vector<int> refs_, level_;
  std::vector<uint32_t> order_;
  std::vector<std::vector<uint32_t>> fanouts_;
  std::vector<char> is_po_;

  void analyse() {
    order_ = live_order(net);
    refs_.assign(net.nodes.size(), 0);
    level_.assign(net.nodes.size(), 0);
    for (uint32_t v : order_) {
      const LNode& l = net.nodes[v];
      int lv = 0;
      for (int k = 0; k < l.n; ++k) {
        ++refs_[l.in[k]];
        lv = std::max(lv, level_[l.in[k]]);
      }
      level_[v] = lv + 1;
    }
    for (uint32_t o : net.outs) ++refs_[o >> 1];
    fanouts_.assign(net.nodes.size(), {});
    is_po_.assign(net.nodes.size(), 0);
    for (uint32_t v : order_)
      for (int k = 0; k < net.nodes[v].n; ++k) {
        auto& fo = fanouts_[net.nodes[v].in[k]];
        if (fo.empty() || fo.back() != v) fo.push_back(v);
      }
    for (uint32_t o : net.outs) is_po_[o >> 1] = 1;
  }

  // maximum fanout-free cone of r (r included)
  void mffc(uint32_t r, std::vector<uint32_t>& cone) {
    cone.clear();
    std::vector<uint32_t> stack{r};
    std::vector<std::pair<uint32_t, int>> undo;
    while (!stack.empty()) {
      const uint32_t v = stack.back();
      stack.pop_back();
      cone.push_back(v);
      const LNode& l = net.nodes[v];
      for (int k = 0; k < l.n; ++k) {
        const uint32_t u = l.in[k];
        if (!net.is_lut(u)) continue;
        undo.push_back({u, 1});
        if (--refs_[u] == 0) stack.push_back(u);
      }
    }
    for (auto& [u, d] : undo) refs_[u] += d;
  }

  static void tt_var(TT& t, int var) {
    for (int w = 0; w < WORDS; ++w) {
      uint64_t x = 0;
      for (int b = 0; b < 64; ++b)
        if (((w * 64 + b) >> var) & 1) x |= 1ull << b;
      t[w] = x;
    }
  }

  // grow a cut from `seed` downwards until `limit` signals (reconvergence-driven)
  std::vector<uint32_t> grow_cut(std::vector<uint32_t> cut, int limit) {
    std::sort(cut.begin(), cut.end());
    cut.erase(std::unique(cut.begin(), cut.end()), cut.end());
    for (int iter = 0; iter < 200; ++iter) {
      int best = -1, best_cost = 1 << 20, best_level = -1;
      for (size_t i = 0; i < cut.size(); ++i) {
        const uint32_t c = cut[i];
        if (!net.is_lut(c)) continue;
        const LNode& l = net.nodes[c];
        int cost = -1;
        for (int k = 0; k < l.n; ++k)
          if (l.in[k] != 0 && !std::binary_search(cut.begin(), cut.end(), l.in[k])) {
            bool dup = false;
            for (int j = 0; j < k; ++j) dup |= l.in[j] == l.in[k];
            if (!dup) ++cost;
          }
        if (cost < best_cost || (cost == best_cost && level_[c] > best_level)) {
          best = int(i);
          best_cost = cost;
          best_level = level_[c];
        }
      }
      if (best < 0 || int(cut.size()) + best_cost > limit) break;
      const LNode l = net.nodes[cut[best]];
      cut.erase(cut.begin() + best);
      for (int k = 0; k < l.n; ++k)
        if (l.in[k] != 0 && !std::binary_search(cut.begin(), cut.end(), l.in[k])) {
          cut.push_back(l.in[k]);
          std::sort(cut.begin(), cut.end());
        }
    }
    return cut;
  }

  struct Div {
    uint32_t id;
    TT t;
  };

  // f constant on every cell of (a, b, c) within care?  returns the LUT table
  static bool fits3(const TT& f, const TT& care, const TT& a, const TT& b, const TT& c, uint8_t* tt_out) {
    uint8_t tt = 0;
    for (int k = 0; k < 8; ++k) {
      bool on = false, off = false;
      for (int w = 0; w < WORDS; ++w) {
        const uint64_t m = ((k & 4) ? a[w] : ~a[w]) & ((k & 2) ? b[w] : ~b[w]) & ((k & 1) ? c[w] : ~c[w]) & care[w];
        if (m & f[w]) on = true;
        if (m & ~f[w]) off = true;
        if (on && off) return false;
      }
      if (on) tt |= uint8_t(1 << k);
    }
    *tt_out = tt;
    return true;
  }


  // A LUT over three of the candidate signals equal to f on care, if any.
  // Filter: sampled (on, off) pattern pairs must each be told apart by one of
  // the three signals before the exact cell check runs.
  template <class Accept>
  bool find_lut3(const TT& f, const TT& care, const std::vector<Div>& win, const std::vector<int>& cand,
                 int ncand, int* ia, int* ib, int* ic, uint8_t* tt, Accept accept) {
    std::vector<int> on, off;
    for (int p = 0; p < (1 << CUT); ++p) {
      if (!((care[p >> 6] >> (p & 63)) & 1)) continue;
      (((f[p >> 6] >> (p & 63)) & 1) ? on : off).push_back(p);
    }
    if (on.empty() || off.empty()) return false;  // constant on care: the caller's wire check covers it
    constexpr int NP = 64;
    int pa[NP], pb[NP];
    uint64_t lcg = 0x9E3779B97F4A7C15ull ^ (uint64_t(on.size()) << 20) ^ off.size();
    for (int i = 0; i < NP; ++i) {
      lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
      pa[i] = on[(lcg >> 33) % on.size()];
      lcg = lcg * 6364136223846793005ull + 1442695040888963407ull;
      pb[i] = off[(lcg >> 33) % off.size()];
    }
    std::vector<uint64_t> dist(ncand, 0);
    for (int d = 0; d < ncand; ++d) {
      const TT& t = win[cand[d]].t;
      uint64_t m = 0;
      for (int i = 0; i < NP; ++i) {
        const int x = int((t[pa[i] >> 6] >> (pa[i] & 63)) & 1), y = int((t[pb[i] >> 6] >> (pb[i] & 63)) & 1);
        if (x != y) m |= 1ull << i;
      }
      dist[d] = m;
    }
    for (int a = 0; a < ncand; ++a)
      for (int b = a + 1; b < ncand; ++b) {
        const uint64_t mab = dist[a] | dist[b];
        for (int c = b + 1; c < ncand; ++c) {
          if ((mab | dist[c]) != ~0ull) continue;
          if (!accept(cand[a], cand[b], cand[c])) continue;
          if (!fits3(f, care, win[cand[a]].t, win[cand[b]].t, win[cand[c]].t, tt)) continue;
          *ia = cand[a];
          *ib = cand[b];
          *ic = cand[c];
          return true;
        }
      }
    return false;
  }

  bool try_root(uint32_t r, bool use_dc, bool two_lut, ResubStats& st) {
    std::vector<uint32_t> cone;
    mffc(r, cone);
    const int k = int(cone.size());
    std::vector<char> in_cone(net.nodes.size(), 0);
    for (uint32_t v : cone) in_cone[v] = 1;
    // leaves of the cone
    std::vector<uint32_t> leaves;
    for (uint32_t v : cone)
      for (int j = 0; j < net.nodes[v].n; ++j)
        if (!in_cone[net.nodes[v].in[j]] && net.nodes[v].in[j] != 0) leaves.push_back(net.nodes[v].in[j]);
    std::sort(leaves.begin(), leaves.end());
    leaves.erase(std::unique(leaves.begin(), leaves.end()), leaves.end());
    if (int(leaves.size()) > CUT) return false;
    // observability window: the fanout of r up to ODC_DEPTH levels; its side
    // inputs join the cut so that the window outputs are functions of the cut
    std::vector<uint32_t> tfo;  // topological (order_) order
    std::vector<uint32_t> seed = leaves;
    if (use_odc_ && !is_po_[r]) {
      // the whole transitive fanout of r: a side input inside it would change
      // with r (and, used as a divisor, close a cycle), so such windows are dropped
      std::vector<char> in_tfo(net.nodes.size(), 0);
      {
        std::vector<uint32_t> stack{r};
        while (!stack.empty()) {
          const uint32_t u = stack.back();
          stack.pop_back();
          for (uint32_t w : fanouts_[u])
            if (!in_tfo[w]) {
              in_tfo[w] = 1;
              stack.push_back(w);
            }
        }
      }
      for (int depth = ODC_DEPTH; depth >= 1; --depth) {
        std::vector<uint32_t> t, frontier{r};
        bool too_big = false;
        for (int dlev = 0; dlev < depth && !too_big; ++dlev) {
          std::vector<uint32_t> next;
          for (uint32_t u : frontier)
            for (uint32_t w : fanouts_[u])
              if (std::find(t.begin(), t.end(), w) == t.end()) {
                t.push_back(w);
                next.push_back(w);
                if (t.size() > 16) too_big = true;
              }
          frontier = next;
        }
        if (too_big) continue;
        std::vector<uint32_t> sd = leaves;
        bool reconverges = false;
        for (uint32_t w : t)
          for (int j = 0; j < net.nodes[w].n; ++j) {
            const uint32_t u = net.nodes[w].in[j];
            if (u != 0 && u != r && std::find(t.begin(), t.end(), u) == t.end() && !in_cone[u]) {
              if (in_tfo[u]) reconverges = true;
              sd.push_back(u);
            }
          }
        if (reconverges) continue;
        std::sort(sd.begin(), sd.end());
        sd.erase(std::unique(sd.begin(), sd.end()), sd.end());
        if (int(sd.size()) > CUT) continue;
        seed = sd;
        for (uint32_t v : order_)
          if (std::find(t.begin(), t.end(), v) != t.end()) tfo.push_back(v);
        break;
      }
    }
    const std::vector<uint32_t> cut = grow_cut(seed, CUT);

    // window: every live node computable from the cut, level <= level(r)
    std::vector<int> slot(net.nodes.size(), -1);
    std::vector<Div> win;
    win.reserve(256);
    for (size_t i = 0; i < cut.size(); ++i) {
      Div d;
      d.id = cut[i];
      tt_var(d.t, int(i));
      slot[cut[i]] = int(win.size());
      win.push_back(d);
    }
    TT zero{};
    auto tt_of = [&](uint32_t u) -> const TT& { return u == 0 ? zero : win[slot[u]].t; };
    int r_slot = -1;
    for (uint32_t v : order_) {
      if (slot[v] >= 0 || refs_[v] == 0) continue;
      if (level_[v] > level_[r]) continue;
      const LNode& l = net.nodes[v];
      bool ok = true;
      for (int j = 0; j < l.n; ++j) ok &= (l.in[j] == 0 || slot[l.in[j]] >= 0);
      if (!ok) continue;
      Div d;
      d.id = v;
      const TT& a = l.n > 0 ? tt_of(l.in[0]) : zero;
      const TT& b = l.n > 1 ? tt_of(l.in[1]) : zero;
      const TT& c = l.n > 2 ? tt_of(l.in[2]) : zero;
      for (int w = 0; w < WORDS; ++w) d.t[w] = lut_eval<uint64_t>(l.tt, a[w], b[w], c[w]);
      slot[v] = int(win.size());
      if (v == r) r_slot = slot[v];
      win.push_back(d);
      if (win.size() > 400) break;
    }
    if (r_slot < 0) return false;
    const TT f = win[r_slot].t;

    // care set over the cut
    TT care;
    const int nvars = int(cut.size());
    for (int w = 0; w < WORDS; ++w) care[w] = ~0ull;
    if (nvars < CUT) {  // unused variables: restrict to their 0 cofactor
      for (int w = 0; w < WORDS; ++w) {
        uint64_t m = 0;
        for (int b = 0; b < 64; ++b)
          if (((w * 64 + b) >> nvars) == 0) m |= 1ull << b;
        care[w] = m;
      }
    }
    if (use_dc) reachable(cut, care);
    if (!tfo.empty()) {
      // window outputs: r's fanout nodes that feed something outside the window
      // (or an output).  Patterns where flipping r changes none of them are
      // don't-cares for r.
      std::vector<TT> v0(tfo.size()), v1(tfo.size());
      auto val = [&](const std::vector<TT>& vv, uint32_t u, bool flip, TT& out) {
        if (u == 0) { out = zero; return; }
        if (u == r) {
          for (int w = 0; w < WORDS; ++w) out[w] = flip ? ~f[w] : f[w];
          return;
        }
        for (size_t i = 0; i < tfo.size(); ++i)
          if (tfo[i] == u) { out = vv[i]; return; }
        out = win[slot[u]].t;
      };
      bool ok = true;
      for (size_t i = 0; i < tfo.size() && ok; ++i) {
        const LNode& l = net.nodes[tfo[i]];
        for (int j = 0; j < l.n; ++j) {
          const uint32_t u = l.in[j];
          if (u != 0 && u != r && std::find(tfo.begin(), tfo.end(), u) == tfo.end() && slot[u] < 0) ok = false;
        }
        if (!ok) break;
        TT a, b, c;
        for (int flip = 0; flip < 2; ++flip) {
          std::vector<TT>& vv = flip ? v1 : v0;
          val(vv, l.n > 0 ? l.in[0] : 0, flip, a);
          val(vv, l.n > 1 ? l.in[1] : 0, flip, b);
          val(vv, l.n > 2 ? l.in[2] : 0, flip, c);
          for (int w = 0; w < WORDS; ++w) vv[i][w] = lut_eval<uint64_t>(l.tt, a[w], b[w], c[w]);
        }
      }
      if (ok) {
        TT obs{};
        bool r_escapes = false;
        for (uint32_t w : fanouts_[r]) r_escapes |= std::find(tfo.begin(), tfo.end(), w) == tfo.end();
        for (size_t i = 0; i < tfo.size(); ++i) {
          bool boundary = is_po_[tfo[i]];
          for (uint32_t w : fanouts_[tfo[i]]) boundary |= std::find(tfo.begin(), tfo.end(), w) == tfo.end();
          if (!boundary) continue;
          for (int w = 0; w < WORDS; ++w) obs[w] |= v0[i][w] ^ v1[i][w];
        }
        if (!r_escapes)
          for (int w = 0; w < WORDS; ++w) care[w] &= obs[w];
      }
    }

    // divisors: window nodes outside the cone (free to use) and, for the LUT
    // moves, the cone's own nodes other than r (using one keeps it and its
    // part of the cone alive, which the gain accounts for)
    std::vector<int> divs, cands;
    for (size_t i = 0; i < win.size(); ++i) {
      if (forbid_ && win[i].id == forbid_) continue;
      if (!in_cone[win[i].id]) divs.push_back(int(i));
      if (win[i].id != r && !(forbid_ && in_cone[win[i].id])) cands.push_back(int(i));
    }
    // cone nodes kept alive by a set of fanins
    auto kept = [&](std::initializer_list<uint32_t> ids) {
      std::vector<uint32_t> stack, seen;
      for (uint32_t u : ids)
        if (in_cone[u]) stack.push_back(u);
      while (!stack.empty()) {
        const uint32_t u = stack.back();
        stack.pop_back();
        if (std::find(seen.begin(), seen.end(), u) != seen.end()) continue;
        seen.push_back(u);
        for (int j = 0; j < net.nodes[u].n; ++j)
          if (in_cone[net.nodes[u].in[j]]) stack.push_back(net.nodes[u].in[j]);
      }
      return int(seen.size());
    };

    // 0 LUTs: an existing signal (or its complement)
    for (int i : divs) {
      bool eq = true, ne = true;
      for (int w = 0; w < WORDS && (eq || ne); ++w) {
        const uint64_t x = (win[i].t[w] ^ f[w]) & care[w];
        if (x) eq = false;
        if (x != care[w]) ne = false;
      }
      if (eq || ne) {
        replace_with_signal(r, win[i].id, ne && !eq);
        ++st.wires;
        return true;
      }
    }
    bool care_empty = true;
    for (int w = 0; w < WORDS; ++w) care_empty &= care[w] == 0;
    if (care_empty) return false;
    if (k - 1 < min_gain_) return false;

    // prefer signals close to r: sort by level descending, keep a bounded set
    std::sort(cands.begin(), cands.end(), [&](int a, int b) {
      const int la = level_[win[a].id], lb = level_[win[b].id];
      return la != lb ? la > lb : win[a].id > win[b].id;
    });
    const int D1 = std::min<int>(int(cands.size()), RESUB_D1);
    // 1 LUT over three signals
    {
      int ia, ib, ic;
      uint8_t tt;
      auto gain1 = [&](int a, int b, int c) {
        return k - 1 - kept({win[a].id, win[b].id, win[c].id}) >= min_gain_;
      };
      if (find_lut3(f, care, win, cands, D1, &ia, &ib, &ic, &tt, gain1)) {
        LNode l;
        l.n = 3;
        l.in[0] = win[ia].id;
        l.in[1] = win[ib].id;
        l.in[2] = win[ic].id;
        l.tt = tt;
        l.tag = net.nodes[r].tag;
        l.ord = net.nodes[r].ord;
        simplify(l);
        net.nodes[r] = l;
        ++st.one;
        return true;
      }
    }
    if (!two_lut || k - 2 < min_gain_) return false;

    // 2 LUTs: f = g(h(a, b, c), d, e).  Within each cell of (d, e), f is 0, 1, h or ~h.
    const int D2 = std::min<int>(int(cands.size()), RESUB_D2);
    const int D3 = std::min<int>(int(cands.size()), RESUB_D3);
    for (int d = 0; d < D2; ++d)
      for (int e = d + 1; e < D2; ++e) {
        const uint32_t did = win[cands[d]].id, eid = win[cands[e]].id;
        if (k - 2 - kept({did, eid}) < min_gain_) continue;
        const TT& td = win[cands[d]].t;
        const TT& te = win[cands[e]].t;
        TT cell[4];
        int kind[4];  // 0 empty, 1 const0, 2 const1, 3 mixed
        int nmixed = 0;
        for (int q = 0; q < 4; ++q) {
          bool on = false, off = false;
          for (int w = 0; w < WORDS; ++w) {
            cell[q][w] = ((q & 2) ? td[w] : ~td[w]) & ((q & 1) ? te[w] : ~te[w]) & care[w];
            if (cell[q][w] & f[w]) on = true;
            if (cell[q][w] & ~f[w]) off = true;
          }
          kind[q] = on && off ? 3 : on ? 2 : off ? 1 : 0;
          nmixed += kind[q] == 3;
        }
        if (nmixed == 0) continue;  // handled by the 1-LUT search
        // polarity of h in the mixed cells (first mixed cell fixed positive)
        int mixed_idx[4], nm = 0;
        for (int q = 0; q < 4; ++q)
          if (kind[q] == 3) mixed_idx[nm++] = q;
        for (int pol = 0; pol < (1 << (nm - 1)); ++pol) {
          TT hf, hcare;
          for (int w = 0; w < WORDS; ++w) hf[w] = hcare[w] = 0;
          for (int i = 0; i < nm; ++i) {
            const int q = mixed_idx[i];
            const bool neg = i > 0 && ((pol >> (i - 1)) & 1);
            for (int w = 0; w < WORDS; ++w) {
              hcare[w] |= cell[q][w];
              hf[w] |= cell[q][w] & (neg ? ~f[w] : f[w]);
            }
          }
          {
            int ia, ib, ic;
            uint8_t th;
            auto gain2 = [&](int a, int b, int c) {
              return k - 2 - kept({win[a].id, win[b].id, win[c].id, did, eid}) >= min_gain_;
            };
            if (find_lut3(hf, hcare, win, cands, D3, &ia, &ib, &ic, &th, gain2)) {
                // g over (h, d, e)
                uint8_t tg = 0;
                for (int q = 0; q < 4; ++q) {
                  // lop3 index: a = h (bit 2), b = d (bit 1), c = e (bit 0)
                  const int dbit = (q >> 1) & 1, ebit = q & 1;
                  for (int hv = 0; hv < 2; ++hv) {
                    int val = 0;
                    if (kind[q] == 2) val = 1;
                    else if (kind[q] == 3) {
                      int i = 0;
                      while (mixed_idx[i] != q) ++i;
                      const bool neg = i > 0 && ((pol >> (i - 1)) & 1);
                      val = neg ? !hv : hv;
                    }
                    if (val) tg |= uint8_t(1 << (hv * 4 + dbit * 2 + ebit));
                  }
                }
                LNode h;
                h.n = 3;
                h.in[0] = win[ia].id;
                h.in[1] = win[ib].id;
                h.in[2] = win[ic].id;
                h.tt = th;
                h.tag = net.nodes[r].tag;
                h.ord = net.nodes[r].ord - 0.5;
                simplify(h);
                net.nodes.push_back(h);
                const uint32_t hid = uint32_t(net.nodes.size() - 1);
                LNode gl;
                gl.n = 3;
                gl.in[0] = hid;
                gl.in[1] = did;
                gl.in[2] = eid;
                gl.tt = tg;
                gl.tag = net.nodes[r].tag;
                gl.ord = net.nodes[r].ord;
                net.nodes[r] = gl;
                ++st.two;
                return true;
            }
          }
        }
      }
    return false;
  }

  // drop inputs the table does not depend on (keeps n and the table consistent)
  static void simplify(LNode& l) {
    for (int k = 0; k < l.n;) {
      const uint8_t m = VAR[k];
      const int sh = 4 >> k;  // distance between the cofactors of variable k
      const uint8_t hi = l.tt & m, lo = l.tt & uint8_t(~m);
      if (uint8_t(hi >> sh) == lo) {
        // independent of input k: remove it, shifting the later inputs up
        uint8_t ntt = 0;
        for (int idx = 0; idx < 8; ++idx) {
          // new assignment idx over inputs (0..n-2 in positions 0..): rebuild old index with var k = 0
          int old = 0, pos = 0;
          for (int j = 0; j < 3; ++j) {
            if (j == k) continue;
            const int bit = (idx >> (2 - pos)) & 1;
            old |= bit << (2 - j);
            ++pos;
          }
          if ((l.tt >> old) & 1) ntt |= uint8_t(1 << idx);
        }
        for (int j = k; j + 1 < 3; ++j) l.in[j] = l.in[j + 1];
        l.in[2] = 0;
        --l.n;
        l.tt = ntt;
      } else {
        ++k;
      }
    }
  }

  // every use of r becomes s (complemented when neg)
  void replace_with_signal(uint32_t r, uint32_t s, bool neg) {
    for (uint32_t v : order_) {
      LNode& l = net.nodes[v];
      for (int k = 0; k < l.n; ++k)
        if (l.in[k] == r) {
          l.in[k] = s;
          if (neg) {
            // complement variable k of the table: swap its cofactors
            const int sh = 4 >> k;
            const uint8_t m = VAR[k];
            l.tt = uint8_t(((l.tt & m) >> sh) | ((l.tt & uint8_t(~m)) << sh));
          }
        }
    }
    for (uint32_t& o : net.outs)
      if ((o >> 1) == r) o = s * 2 + ((o & 1) ^ (neg ? 1 : 0));
  }

  // care &= { cut assignments produced by some assignment of a deeper cut }
  void reachable(const std::vector<uint32_t>& cut, TT& care) {
    std::vector<uint32_t> deep = grow_cut(cut, DEEP);
    if (deep == cut) return;
    const int nv = int(deep.size());
    const size_t W = nv <= 6 ? 1 : (size_t(1) << (nv - 6));
    // nodes between deep and cut, topological
    std::vector<int> slot(net.nodes.size(), -1);
    std::vector<std::vector<uint64_t>> val;
    auto var_words = [&](int var) {
      std::vector<uint64_t> t(W);
      for (size_t w = 0; w < W; ++w) {
        uint64_t x = 0;
        if (var < 6) {
          static const uint64_t pat[6] = {0xAAAAAAAAAAAAAAAAull, 0xCCCCCCCCCCCCCCCCull, 0xF0F0F0F0F0F0F0F0ull,
                                          0xFF00FF00FF00FF00ull, 0xFFFF0000FFFF0000ull, 0xFFFFFFFF00000000ull};
          x = pat[var];
        } else {
          x = ((w >> (var - 6)) & 1) ? ~0ull : 0ull;
        }
        t[w] = x;
      }
      return t;
    };
    for (size_t i = 0; i < deep.size(); ++i) {
      slot[deep[i]] = int(val.size());
      val.push_back(var_words(int(i)));
    }
    std::vector<uint64_t> zero(W, 0);
    // only the transitive fanin of the cut, bounded by the deep cut
    std::vector<char> need(net.nodes.size(), 0);
    {
      std::vector<uint32_t> stack(cut.begin(), cut.end());
      while (!stack.empty()) {
        const uint32_t v = stack.back();
        stack.pop_back();
        if (need[v] || slot[v] >= 0 || !net.is_lut(v)) continue;
        need[v] = 1;
        for (int j = 0; j < net.nodes[v].n; ++j) stack.push_back(net.nodes[v].in[j]);
      }
    }
    int missing = 0;
    for (uint32_t c : cut) missing += slot[c] < 0;
    for (uint32_t v : order_) {
      if (missing == 0) break;
      if (!need[v] || slot[v] >= 0) continue;
      const LNode& l = net.nodes[v];
      bool ok = true;
      for (int j = 0; j < l.n; ++j) ok &= (l.in[j] == 0 || slot[l.in[j]] >= 0);
      if (!ok) return;  // a fanin outside the deep cut: should not happen
      std::vector<uint64_t> t(W);
      const std::vector<uint64_t>& a = (l.n > 0 && l.in[0]) ? val[slot[l.in[0]]] : zero;
      const std::vector<uint64_t>& b = (l.n > 1 && l.in[1]) ? val[slot[l.in[1]]] : zero;
      const std::vector<uint64_t>& c = (l.n > 2 && l.in[2]) ? val[slot[l.in[2]]] : zero;
      for (size_t w = 0; w < W; ++w) t[w] = lut_eval<uint64_t>(l.tt, a[w], b[w], c[w]);
      slot[v] = int(val.size());
      val.push_back(std::move(t));
      if (std::find(cut.begin(), cut.end(), v) != cut.end()) --missing;
    }
    if (missing) return;  // should not happen
    TT seen{};
    const size_t npat = size_t(1) << nv;
    std::vector<const uint64_t*> cv;
    for (uint32_t c : cut) cv.push_back(val[slot[c]].data());
    for (size_t p = 0; p < npat; ++p) {
      uint32_t idx = 0;
      for (size_t i = 0; i < cv.size(); ++i) idx |= uint32_t((cv[i][p >> 6] >> (p & 63)) & 1) << i;
      seen[idx >> 6] |= 1ull << (idx & 63);
    }
    for (int w = 0; w < WORDS; ++w) care[w] &= seen[w];
  }
};

// The whole post-mapping flow on one network: resubstitution to a fixed point,
// then node elimination and resubstitution in turn while LUTs still disappear.
inline void optimize_net(LutNet& net, int rounds = 4) {
  Resub(net).run(4);
  for (int it = 0; it < rounds; ++it) {
    const int removed = Resub(net).eliminate();
    Resub(net).run(4);
    if (removed == 0) break;
  }
}

// Straight-line device code for a LUT network (see lutmap::emit).
inline std::string emit_net(const LutNet& net, const std::vector<std::string>& input_names,
                            const std::vector<std::string>& output_names) {
  std::string s;
  std::vector<std::string> name(net.nodes.size());
  name[0] = "0u";
  for (uint32_t i = 1; i <= net.n_pi; ++i) name[i] = input_names[i - 1];
  const auto order = natural_order(net);
  std::vector<int> lut_uses(net.nodes.size(), 0), pos_out(net.nodes.size(), 0), neg_out(net.nodes.size(), 0);
  for (uint32_t v : order)
    for (int k = 0; k < net.nodes[v].n; ++k) ++lut_uses[net.nodes[v].in[k]];
  for (uint32_t o : net.outs) ((o & 1) ? neg_out : pos_out)[o >> 1]++;
  std::vector<char> flipped(net.nodes.size(), 0);
  char buf[256];
  uint32_t serial = 0;
  for (uint32_t v : order) {
    const LNode& l = net.nodes[v];
    uint8_t tt = l.tt;
    if (lut_uses[v] == 0 && pos_out[v] == 0 && neg_out[v] > 0) {
      tt = uint8_t(~tt);
      flipped[v] = 1;
    }
    std::string ops[3] = {"0u", "0u", "0u"};
    for (int k = 0; k < l.n; ++k) ops[k] = name[l.in[k]];
    name[v] = "t" + std::to_string(++serial);
    std::snprintf(buf, sizeof buf, "    const w32 %s = lop3<0x%02X>(%s, %s, %s);\n", name[v].c_str(), tt,
                  ops[0].c_str(), ops[1].c_str(), ops[2].c_str());
    s += buf;
  }
  for (size_t i = 0; i < net.outs.size(); ++i) {
    const uint32_t o = net.outs[i], v = o >> 1;
    std::string e;
    if (v == 0) e = (o & 1) ? "ONES" : "0u";
    else if (flipped[v]) e = name[v];
    else e = (o & 1) ? ("~" + name[v]) : name[v];
    s += "    " + output_names[i] + " = " + e + ";\n";
  }
  return s;
}

}  // namespace lutmap

namespace lutmap {

// The LUT network as an AND/XOR graph again (Shannon expansion of every table,
// XOR forms detected), so that the structural mapper can look for covers whose
// LUT boundaries differ from the network's own.
inline Lit graph_of_table(Graph& g, uint8_t tt, Lit a, Lit b, Lit c) {
  auto two = [&](uint8_t t4, Lit x, Lit y) -> Lit {  // 2-input table over (x, y): bit index x*2 + y
    switch (t4 & 15) {
      case 0x0: return 0;
      case 0xF: return 1;
      case 0xC: return x;
      case 0x3: return x ^ 1;
      case 0xA: return y;
      case 0x5: return y ^ 1;
      case 0x6: return g.XOR(x, y);
      case 0x9: return g.XOR(x, y) ^ 1;
      default: break;
    }
    // AND-type: exactly one or three minterms
    Lit r = 0;
    bool first = true;
    int ones = 0;
    for (int k = 0; k < 4; ++k) ones += (t4 >> k) & 1;
    const uint8_t t = ones == 1 ? t4 : uint8_t(~t4 & 15);
    for (int k = 0; k < 4; ++k)
      if ((t >> k) & 1) {
        const Lit m = g.AND((k & 2) ? x : (x ^ 1), (k & 1) ? y : (y ^ 1));
        r = first ? m : g.OR(r, m);
        first = false;
      }
    return ones == 1 ? r : (r ^ 1);
  };
  const uint8_t f1 = (tt >> 4) & 15, f0 = tt & 15;  // cofactors of a over (b, c)
  if (f1 == f0) return two(f0, b, c);
  if (f1 == uint8_t(~f0 & 15)) return g.XOR(a, two(f0, b, c));
  const Lit h1 = two(f1, b, c), h0 = two(f0, b, c);
  return g.OR(g.AND(a, h1), g.AND(a ^ 1, h0));
}

inline std::vector<Lit> to_graph(const LutNet& net, Graph& g) {
  std::vector<Lit> lit(net.nodes.size(), 0);
  for (uint32_t i = 1; i <= net.n_pi; ++i) lit[i] = g.input();
  g.tag.resize(g.nodes.size(), 0);
  for (uint32_t v : natural_order(net)) {
    const LNode& l = net.nodes[v];
    g.cur = l.tag;
    lit[v] = graph_of_table(g, l.tt, l.n > 0 ? lit[l.in[0]] : 0, l.n > 1 ? lit[l.in[1]] : 0,
                            l.n > 2 ? lit[l.in[2]] : 0);
  }
  std::vector<Lit> outs;
  for (uint32_t o : net.outs) outs.push_back(lit[o >> 1] ^ (o & 1));
  return outs;
}

}  // namespace lutmap

namespace lutmap {

// The complete flow behind the generated covers: structural cover of the
// template graph -> optimize_net -> re-map the optimised network (its LUT
// boundaries give the structural mapper new choices) and optimise again, while
// the network still shrinks.  graph() is left pointing at g.
inline LutNet optimised_cover(Graph& g, const std::vector<Lit>& outs, bool optimise = true) {
  auto M = map_luts(g, outs);
  recover_area(g, M, outs);
  LutNet net = from_mapping(g, M, outs);
  if (!optimise) return net;
  optimize_net(net);
  size_t best = count_luts(net);
  for (int it = 0; it < 3; ++it) {
    Graph g2;
    g2.stage_names = g.stage_names;
    graph() = &g2;
    const std::vector<Lit> o2 = to_graph(net, g2);
    auto M2 = map_luts(g2, o2);
    recover_area(g2, M2, o2);
    LutNet n2 = from_mapping(g2, M2, o2);
    optimize_net(n2);
    graph() = &g;
    const size_t n = count_luts(n2);
    if (n >= best) break;
    best = n;
    net = n2;
  }
  return net;
}

}  // namespace lutmap

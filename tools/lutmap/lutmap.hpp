// tools/lutmap/lutmap.hpp -- build-time LOP3 technology mapper.
//
// The bitslice networks (paper_1602_04716_b200/csrc/bfp_circuits.cuh) are
// evaluated on a symbolic word `Sym`: every & | ^ ~ builds a node of a
// hash-consed AND/XOR graph with complemented edges and constant folding.
// The graph is then covered with 3-input LUTs (one LOP3.LUT each on sm_100a)
// by priority-cut enumeration (K = 3, area flow, then exact-area recovery
// passes), and emitted as straight-line lop3.b32 device code.  ptxas keeps
// pinned lop3.b32 one-for-one, so the SASS LOP3 count equals the mapped count.
#pragma once

#include <algorithm>
#include <array>
#include <cstdint>
#include <cstdio>
#include <string>
#include <unordered_map>
#include <vector>

namespace lutmap {

// literal = node * 2 + complement; node 0 is the constant 0 (lit 0 = 0, lit 1 = 1)
using Lit = uint32_t;

struct Node {
  uint8_t kind;  // 0 const, 1 input, 2 and, 3 xor
  Lit a, b;
};

struct Graph {
  std::vector<Node> nodes{Node{0, 0, 0}};
  std::unordered_map<uint64_t, uint32_t> hash;
  uint32_t n_inputs = 0;
  // stage of the template code that created each node (BFP_STAGE markers;
  // the per-stage LUT report of tools/lutmap/stages.cpp)
  std::vector<uint16_t> tag{0};
  std::vector<std::string> stage_names{"(inputs)"};
  uint16_t cur = 0;
  void stage(const char* name) {
    for (size_t i = 0; i < stage_names.size(); ++i)
      if (stage_names[i] == name) {
        cur = uint16_t(i);
        return;
      }
    stage_names.push_back(name);
    cur = uint16_t(stage_names.size() - 1);
  }

  Lit input() {
    nodes.push_back(Node{1, 0, 0});
    tag.push_back(0);
    ++n_inputs;
    return Lit(nodes.size() - 1) * 2;
  }
  Lit mk(uint8_t kind, Lit a, Lit b) {
    if (a > b) std::swap(a, b);
    const uint64_t key = (uint64_t(kind) << 62) | (uint64_t(a) << 31) | b;
    auto it = hash.find(key);
    if (it != hash.end()) return Lit(it->second) * 2;
    nodes.push_back(Node{kind, a, b});
    tag.push_back(cur);
    hash.emplace(key, uint32_t(nodes.size() - 1));
    return Lit(nodes.size() - 1) * 2;
  }
  Lit AND(Lit a, Lit b) {
    if (a == 0 || b == 0) return 0;
    if (a == 1) return b;
    if (b == 1) return a;
    if (a == b) return a;
    if ((a ^ b) == 1) return 0;
    return mk(2, a, b);
  }
  Lit XOR(Lit a, Lit b) {
    Lit c = (a & 1) ^ (b & 1);
    a &= ~1u;
    b &= ~1u;
    if (a == 0) return b ^ c;
    if (b == 0) return a ^ c;
    if (a == b) return c;
    return mk(3, a, b) ^ c;
  }
  Lit OR(Lit a, Lit b) { return AND(a ^ 1, b ^ 1) ^ 1; }
};

inline Graph*& graph() {
  static Graph* g = nullptr;
  return g;
}

struct Sym {
  Lit l = 0;
  Sym() = default;
  Sym(uint32_t c) : l(c ? 1 : 0) {}  // only 0 and all-ones constants occur
  static Sym of(Lit x) {
    Sym s;
    s.l = x;
    return s;
  }
  friend Sym operator&(Sym a, Sym b) { return of(graph()->AND(a.l, b.l)); }
  friend Sym operator|(Sym a, Sym b) { return of(graph()->OR(a.l, b.l)); }
  friend Sym operator^(Sym a, Sym b) { return of(graph()->XOR(a.l, b.l)); }
  friend Sym operator~(Sym a) { return of(a.l ^ 1); }
  Sym& operator&=(Sym b) { return *this = *this & b; }
  Sym& operator|=(Sym b) { return *this = *this | b; }
  Sym& operator^=(Sym b) { return *this = *this ^ b; }
};

// ------------------------------------------------------------------ mapper
struct Cut {
  uint8_t n = 0;
  uint32_t leaf[3] = {0, 0, 0};  // node ids, sorted
  uint8_t tt = 0;                // function over leaves (leaf0 -> 0xF0 ... as lop3 a,b,c)
  float af = 0;
};

// truth-table variable masks for leaf positions 0, 1, 2 = lop3 inputs a, b, c
constexpr uint8_t VAR[3] = {0xF0, 0xCC, 0xAA};

struct Mapping {
  std::vector<int> best;                 // chosen cut index per node
  std::vector<std::vector<Cut>> cuts;    // per node
  std::vector<uint32_t> required;        // node ids that become LUTs (topological)
  size_t luts = 0;
};

// expand tt over cut `c` to the leaf set `m` (c.leaf subset of m.leaf)
inline uint8_t expand(const Cut& c, const Cut& m) {
  uint8_t out = 0;
  for (int k = 0; k < 8; ++k) {
    // assignment k over m's leaves: bit i of the assignment = value of m.leaf[i]
    // where the variable mask VAR[i] has bit k set
    int idx = 0;
    for (int j = 0; j < c.n; ++j) {
      int pos = 0;
      while (m.leaf[pos] != c.leaf[j]) ++pos;
      if ((VAR[pos] >> k) & 1) idx |= 1 << (2 - j);  // c's variable j -> lop3 bit (2 - j)
    }
    // evaluate c.tt at c-assignment idx (bit index: a*4 + b*2 + c)
    if ((c.tt >> idx) & 1) out |= uint8_t(1 << k);
  }
  return out;
}

inline bool merge(const Cut& x, const Cut& y, Cut& m) {
  uint32_t buf[6];
  int n = 0;
  int i = 0, j = 0;
  while (i < x.n || j < y.n) {
    uint32_t v;
    if (j >= y.n || (i < x.n && x.leaf[i] < y.leaf[j])) v = x.leaf[i++];
    else if (i >= x.n || y.leaf[j] < x.leaf[i]) v = y.leaf[j++];
    else { v = x.leaf[i++]; ++j; }
    if (n == 3) return false;
    buf[n++] = v;
  }
  m.n = uint8_t(n);
  for (int k = 0; k < n; ++k) m.leaf[k] = buf[k];
  return true;
}

inline Mapping map_luts(const Graph& g, const std::vector<Lit>& outputs, int passes = 4,
                        size_t max_cuts = 10) {
  const size_t N = g.nodes.size();
  Mapping M;
  M.cuts.assign(N, {});
  M.best.assign(N, 0);
  std::vector<float> refs(N, 1.0f), af_best(N, 0.0f);
  // initial fanout estimate
  {
    std::vector<int> fo(N, 0);
    for (size_t v = 1; v < N; ++v) {
      const Node& nd = g.nodes[v];
      if (nd.kind >= 2) {
        ++fo[nd.a >> 1];
        ++fo[nd.b >> 1];
      }
    }
    for (Lit o : outputs) ++fo[o >> 1];
    for (size_t v = 0; v < N; ++v) refs[v] = std::max(1, fo[v]);
  }
  for (int pass = 0; pass < passes; ++pass) {
    for (size_t v = 1; v < N; ++v) {
      const Node& nd = g.nodes[v];
      auto& cs = M.cuts[v];
      cs.clear();
      if (nd.kind == 1) {
        Cut t;
        t.n = 1;
        t.leaf[0] = uint32_t(v);
        t.tt = VAR[0];
        t.af = 0;
        cs.push_back(t);
        af_best[v] = 0;
        continue;
      }
      const uint32_t va = nd.a >> 1, vb = nd.b >> 1;
      const bool ca = nd.a & 1, cb = nd.b & 1;
      auto child_cuts = [&](uint32_t u) {
        std::vector<Cut> r = M.cuts[u];
        if (g.nodes[u].kind >= 2) {  // the trivial cut {u}
          Cut t;
          t.n = 1;
          t.leaf[0] = u;
          t.tt = VAR[0];
          r.push_back(t);
        }
        return r;
      };
      const std::vector<Cut> A = child_cuts(va), B = child_cuts(vb);
      std::vector<Cut> cand;
      for (const Cut& x : A)
        for (const Cut& y : B) {
          Cut m;
          if (!merge(x, y, m)) continue;
          uint8_t tx = expand(x, m), ty = expand(y, m);
          if (ca) tx = uint8_t(~tx);
          if (cb) ty = uint8_t(~ty);
          m.tt = nd.kind == 2 ? uint8_t(tx & ty) : uint8_t(tx ^ ty);
          float af = 1.0f;
          for (int k = 0; k < m.n; ++k) {
            const uint32_t l = m.leaf[k];
            if (g.nodes[l].kind >= 2) af += af_best[l] / refs[l];
          }
          m.af = af;
          bool dup = false;
          for (const Cut& c : cand)
            if (c.n == m.n && std::equal(c.leaf, c.leaf + c.n, m.leaf)) { dup = true; break; }
          if (!dup) cand.push_back(m);
        }
      std::sort(cand.begin(), cand.end(), [](const Cut& p, const Cut& q) {
        return p.af != q.af ? p.af < q.af : p.n < q.n;
      });
      if (cand.size() > max_cuts) cand.resize(max_cuts);
      cs = cand;
      M.best[v] = 0;
      af_best[v] = cs.empty() ? 1e9f : cs[0].af;
    }
    // derive the cover from the outputs; update reference counts
    std::vector<int> used(N, 0);
    std::vector<uint32_t> stack;
    for (Lit o : outputs) {
      const uint32_t v = o >> 1;
      if (g.nodes[v].kind >= 2) stack.push_back(v);
    }
    std::vector<char> seen(N, 0);
    M.required.clear();
    while (!stack.empty()) {
      const uint32_t v = stack.back();
      stack.pop_back();
      if (seen[v]) continue;
      seen[v] = 1;
      M.required.push_back(v);
      const Cut& c = M.cuts[v][0];
      for (int k = 0; k < c.n; ++k) {
        ++used[c.leaf[k]];
        if (g.nodes[c.leaf[k]].kind >= 2 && !seen[c.leaf[k]]) stack.push_back(c.leaf[k]);
      }
    }
    for (Lit o : outputs) ++used[o >> 1];
    for (size_t v = 0; v < N; ++v) refs[v] = 0.5f * refs[v] + 0.5f * std::max(1, used[v]);
    std::sort(M.required.begin(), M.required.end());
    M.luts = M.required.size();
  }
  return M;
}

// Exact-area recovery (reference/dereference of maximum fanout-free cones):
// for every node of the cover, pick the cut whose cone adds the fewest LUTs
// given the rest of the cover.
struct AreaRecovery {
  const Graph& g;
  Mapping& M;
  std::vector<int> refs;
  AreaRecovery(const Graph& g_, Mapping& M_) : g(g_), M(M_), refs(g_.nodes.size(), 0) {}
  bool internal(uint32_t v) const { return g.nodes[v].kind >= 2; }
  int deref(uint32_t v, const Cut& c) {
    int area = 1;
    for (int k = 0; k < c.n; ++k) {
      const uint32_t l = c.leaf[k];
      if (internal(l) && --refs[l] == 0) area += deref(l, M.cuts[l][M.best[l]]);
    }
    return area;
  }
  int ref(uint32_t v, const Cut& c) {
    int area = 1;
    for (int k = 0; k < c.n; ++k) {
      const uint32_t l = c.leaf[k];
      if (internal(l) && refs[l]++ == 0) area += ref(l, M.cuts[l][M.best[l]]);
    }
    return area;
  }
  void run(const std::vector<Lit>& outputs, int passes) {
    for (Lit o : outputs)
      if (internal(o >> 1) && refs[o >> 1]++ == 0) ref(o >> 1, M.cuts[o >> 1][M.best[o >> 1]]);
    for (int p = 0; p < passes; ++p) {
      for (size_t v = 1; v < g.nodes.size(); ++v) {
        if (!internal(uint32_t(v)) || refs[v] == 0) continue;
        auto& cs = M.cuts[v];
        deref(uint32_t(v), cs[M.best[v]]);
        int best = M.best[v], best_area = 1 << 30;
        for (size_t i = 0; i < cs.size(); ++i) {
          const int a = ref(uint32_t(v), cs[i]);
          deref(uint32_t(v), cs[i]);
          if (a < best_area) {
            best_area = a;
            best = int(i);
          }
        }
        M.best[v] = best;
        ref(uint32_t(v), cs[best]);
      }
    }
    M.required.clear();
    for (size_t v = 1; v < g.nodes.size(); ++v)
      if (internal(uint32_t(v)) && refs[v] > 0) M.required.push_back(uint32_t(v));
    M.luts = M.required.size();
  }
};

inline void recover_area(const Graph& g, Mapping& M, const std::vector<Lit>& outputs, int passes = 3) {
  AreaRecovery r(g, M);
  r.run(outputs, passes);
}

// Straight-line device code for the cover.  A complemented output whose LUT
// feeds nothing else gets the complemented table instead of an extra NOT.
inline std::string emit(const Graph& g, const Mapping& M, const std::vector<std::string>& input_names,
                        const std::vector<Lit>& outputs, const std::vector<std::string>& output_names) {
  std::string s;
  const size_t N = g.nodes.size();
  std::vector<std::string> name(N);
  uint32_t in = 0;
  for (size_t v = 1; v < N; ++v)
    if (g.nodes[v].kind == 1) name[v] = input_names[in++];
  std::vector<int> lut_uses(N, 0), pos_out(N, 0), neg_out(N, 0);
  for (uint32_t v : M.required) {
    const Cut& c = M.cuts[v][M.best[v]];
    for (int k = 0; k < c.n; ++k) ++lut_uses[c.leaf[k]];
  }
  for (Lit o : outputs) ((o & 1) ? neg_out : pos_out)[o >> 1]++;
  std::vector<char> flipped(N, 0);
  char buf[256];
  for (uint32_t v : M.required) {
    const Cut& c = M.cuts[v][M.best[v]];
    uint8_t tt = c.tt;
    if (lut_uses[v] == 0 && pos_out[v] == 0 && neg_out[v] > 0) {
      tt = uint8_t(~tt);
      flipped[v] = 1;
    }
    std::string ops[3] = {"0u", "0u", "0u"};
    for (int k = 0; k < c.n; ++k) ops[k] = name[c.leaf[k]];
    std::snprintf(buf, sizeof buf, "    const w32 t%u = lop3<0x%02X>(%s, %s, %s);\n", v, tt,
                  ops[0].c_str(), ops[1].c_str(), ops[2].c_str());
    s += buf;
    name[v] = "t" + std::to_string(v);
  }
  for (size_t i = 0; i < outputs.size(); ++i) {
    const Lit o = outputs[i];
    const uint32_t v = o >> 1;
    std::string e;
    if (v == 0) e = (o & 1) ? "ONES" : "0u";
    else if (flipped[v]) e = name[v];
    else e = (o & 1) ? ("~" + name[v]) : name[v];
    s += "    " + output_names[i] + " = " + e + ";\n";
  }
  return s;
}

}  // namespace lutmap

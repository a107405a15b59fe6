// Host-side graph ingest: make_graph validation and the GroupedGraph
// transforms (colocation, co-placement, fusion), restated in C++17 for the
// C ABI (bx_grouped_*). The placement hot path runs on the GPU; this is the
// ingest that feeds it, sequential by nature (fusion is order-dependent,
// SURVEY.md finding 6), so it stays on the host as the north star asks.
//
// Semantics follow the reference exactly:
//   make_graph           proj/src/graph.cpp:99-194 (validation order and texts)
//   singleton_groups     proj/src/transforms.cpp:300-327
//   apply_colocation     proj/src/transforms.cpp:329-351
//   apply_coplacement    proj/src/transforms.cpp:353-388
//   fuse_operators       proj/src/transforms.cpp:390-444
//   GroupMerger          proj/src/transforms.cpp:23-244
// Outputs are canonical — meta nodes numbered by ascending smallest base
// member, edges sorted by (src, dst) — so the union-find's choice of
// surviving root never shows; this implementation keeps flat arrays and
// epoch-stamped DFS instead of std::set / std::map where order is not
// observable.
#include <algorithm>
#include <climits>
#include <cstdint>
#include <cstring>
#include <map>
#include <numeric>
#include <queue>
#include <stdexcept>
#include <string>
#include <unordered_map>
#include <vector>

#include "../../include/baechi_b200.h"

namespace {

struct VErr : std::runtime_error {
  explicit VErr(const std::string &m) : std::runtime_error(m) {}
};

struct Base {
  int n = 0;
  std::vector<int64_t> id, k, temp, perm, out;
  std::vector<int32_t> label;    // colocation label or -1
  std::vector<int64_t> pair;     // coplace peer id
  std::vector<uint8_t> has_pair;
  std::vector<int32_t> esrc, edst;  // dense indices, sorted (src, dst)
  std::vector<int64_t> ebytes;
  int index_of(int64_t x) const {
    auto it = std::lower_bound(id.begin(), id.end(), x);
    if (it == id.end() || *it != x) throw VErr("dangling reference: unknown node id " + std::to_string(x));
    return static_cast<int>(it - id.begin());
  }
};

struct Meta {  // a GroupedGraph
  std::vector<std::vector<int>> members;
  std::vector<int64_t> k, temp, perm, out;
  std::vector<int32_t> esrc, edst, ecount;
  std::vector<int64_t> ebytes;
  std::vector<int32_t> group_of;
  int V() const { return static_cast<int>(members.size()); }
};

// make_graph (graph.cpp:99-194)
Base make_graph(const bx_base_graph &in) {
  Base g;
  const int n = in.nodes;
  std::vector<int> ord(n);
  std::iota(ord.begin(), ord.end(), 0);
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return in.id[a] < in.id[b]; });
  g.n = n;
  for (int r = 0; r < n; ++r) {
    int i = ord[r];
    if (r > 0 && in.id[i] == g.id.back()) throw VErr("duplicate node id " + std::to_string(in.id[i]));
    g.id.push_back(in.id[i]);
    g.k.push_back(in.compute_us[i]);
    g.temp.push_back(in.temp_bytes[i]);
    g.perm.push_back(in.perm_bytes[i]);
    g.out.push_back(in.out_bytes[i]);
    g.label.push_back(in.coloc_label ? in.coloc_label[i] : -1);
    bool hp = in.has_pair && in.has_pair[i];
    g.has_pair.push_back(hp);
    g.pair.push_back(hp ? in.coplace_peer[i] : 0);
  }
  for (int i = 0; i < n; ++i)
    if (g.k[i] < 0 || g.temp[i] < 0 || g.perm[i] < 0 || g.out[i] < 0)
      throw VErr("node " + std::to_string(g.id[i]) + " has a negative field");
  for (int i = 0; i < n; ++i) {
    if (!g.has_pair[i]) continue;
    int64_t peer = g.pair[i];
    if (peer == g.id[i]) throw VErr("node " + std::to_string(g.id[i]) + " coplace_pair references itself");
    int p = g.index_of(peer);
    if (!g.has_pair[p] || g.pair[p] != g.id[i])
      throw VErr("coplace_pair between " + std::to_string(g.id[i]) + " and " + std::to_string(peer) +
                 " is not symmetric");
  }
  std::vector<std::pair<int, int>> es;
  std::vector<int64_t> eb;
  for (int e = 0; e < in.edges; ++e) {
    if (in.tensor_bytes[e] < 0)
      throw VErr("edge " + std::to_string(in.src[e]) + "->" + std::to_string(in.dst[e]) + " has negative bytes");
    if (in.src[e] == in.dst[e]) throw VErr("self edge on node " + std::to_string(in.src[e]));
    int s = g.index_of(in.src[e]);
    int d = g.index_of(in.dst[e]);
    es.push_back({s, d});
    eb.push_back(in.tensor_bytes[e]);
  }
  std::vector<int> eo(es.size());
  std::iota(eo.begin(), eo.end(), 0);
  std::stable_sort(eo.begin(), eo.end(), [&](int a, int b) { return es[a] < es[b]; });
  for (size_t r = 0; r < eo.size(); ++r) {
    const auto &cur = es[eo[r]];
    if (r > 0 && cur == es[eo[r - 1]])
      throw VErr("duplicate edge " + std::to_string(g.id[cur.first]) + "->" + std::to_string(g.id[cur.second]));
    g.esrc.push_back(cur.first);
    g.edst.push_back(cur.second);
    g.ebytes.push_back(eb[eo[r]]);
  }
  // acyclicity (Kahn, smallest index first); leftovers lie on a cycle
  const int E = static_cast<int>(g.esrc.size());
  std::vector<int> out_off(n + 1, 0), indeg(n, 0);
  for (int e = 0; e < E; ++e) {
    out_off[g.esrc[e] + 1]++;
    indeg[g.edst[e]]++;
  }
  for (int v = 0; v < n; ++v) out_off[v + 1] += out_off[v];
  std::priority_queue<int, std::vector<int>, std::greater<int>> ready;
  for (int v = 0; v < n; ++v)
    if (!indeg[v]) ready.push(v);
  int seen = 0;
  while (!ready.empty()) {
    int u = ready.top();
    ready.pop();
    ++seen;
    for (int e = out_off[u]; e < out_off[u + 1]; ++e)
      if (--indeg[g.edst[e]] == 0) ready.push(g.edst[e]);
  }
  if (seen != n) {
    // extract_cycle (graph.cpp:52-84): from the first leftover node, follow
    // the first out-edge that stays among leftovers until a node repeats
    int cur = 0;
    while (indeg[cur] == 0) ++cur;
    std::vector<int> path, pos(n, -1);
    while (pos[cur] < 0) {
      pos[cur] = static_cast<int>(path.size());
      path.push_back(cur);
      int next = -1;
      for (int e = out_off[cur]; e < out_off[cur + 1]; ++e)
        if (indeg[g.edst[e]] > 0) {
          next = g.edst[e];
          break;
        }
      cur = next;
    }
    std::string m = "graph has a cycle through node ids {";
    for (size_t i = pos[cur]; i < path.size(); ++i) m += (i > size_t(pos[cur]) ? ", " : "") + std::to_string(g.id[path[i]]);
    throw VErr(m + "}");
  }
  return g;
}

Meta singleton_groups(const Base &b) {
  Meta m;
  m.members.resize(b.n);
  for (int i = 0; i < b.n; ++i) m.members[i] = {i};
  m.k = b.k;
  m.temp = b.temp;
  m.perm = b.perm;
  m.out = b.out;
  m.esrc = b.esrc;
  m.edst = b.edst;
  m.ebytes = b.ebytes;
  m.ecount.assign(b.esrc.size(), 1);
  m.group_of.resize(b.n);
  std::iota(m.group_of.begin(), m.group_of.end(), 0);
  return m;
}

// GroupMerger (transforms.cpp:23-244): union-find over an input grouping's
// meta nodes with aggregated adjacency between live roots.
class Merger {
 public:
  struct Agg {
    int64_t bytes = 0;
    int count = 0;
  };
  // levels: with `track_levels` (merges that keep the meta graph acyclic:
  // co-placement and fusion) every live root carries a topological potential
  // lvl(u) < lvl(v) for every edge u -> v, kept valid across merges; a path
  // search toward b then never enters a root with lvl >= lvl(b).
  explicit Merger(const Meta &in, bool track_levels = false) : in_(in), track_(track_levels) {
    const int n = in.V();
    parent_.resize(n);
    minm_.resize(n);
    succ_.resize(n);
    pred_.resize(n);
    out_base_.assign(n, 0);
    in_base_.assign(n, 0);
    stamp_.assign(n, 0);
    for (int g = 0; g < n; ++g) {
      parent_[g] = g;
      minm_[g] = in.members[g].front();
    }
    for (size_t e = 0; e < in.esrc.size(); ++e) {
      int s = in.esrc[e], d = in.edst[e];
      succ_[s][d] = Agg{in.ebytes[e], in.ecount[e]};
      pred_[d][s] = Agg{in.ebytes[e], in.ecount[e]};
      out_base_[s] += in.ecount[e];
      in_base_[d] += in.ecount[e];
    }
    if (track_) {  // longest-path levels (Kahn); a cyclic input disables pruning
      lvl_.assign(n, 0);
      std::vector<int> indeg(n, 0), q;
      for (int g = 0; g < n; ++g) indeg[g] = static_cast<int>(pred_[g].size());
      for (int g = 0; g < n; ++g)
        if (!indeg[g]) q.push_back(g);
      for (size_t h = 0; h < q.size(); ++h)
        for (const auto &kv : succ_[q[h]]) {
          lvl_[kv.first] = std::max(lvl_[kv.first], lvl_[q[h]] + 1);
          if (--indeg[kv.first] == 0) q.push_back(kv.first);
        }
      if (static_cast<int>(q.size()) != n) track_ = false;
    }
  }
  int find(int g) {
    while (parent_[g] != g) {
      parent_[g] = parent_[parent_[g]];
      g = parent_[g];
    }
    return g;
  }
  int out_base(int r) const { return out_base_[r]; }
  int in_base(int r) const { return in_base_[r]; }

  int unite(int x, int y) {
    int a = find(x), b = find(y);
    if (a == b) return a;
    int s = a, l = b;
    if (succ_[s].size() + pred_[s].size() < succ_[l].size() + pred_[l].size()) std::swap(s, l);
    minm_[s] = std::min(minm_[s], minm_[l]);
    auto it = succ_[s].find(l);
    if (it != succ_[s].end()) {  // s -> l becomes internal
      out_base_[s] -= it->second.count;
      succ_[s].erase(it);
      pred_[l].erase(s);
    }
    it = pred_[s].find(l);
    if (it != pred_[s].end()) {  // l -> s becomes internal
      in_base_[s] -= it->second.count;
      pred_[s].erase(it);
      succ_[l].erase(s);
    }
    for (const auto &kv : succ_[l]) {
      const int t = kv.first;
      Agg &slot = succ_[s][t];
      slot.bytes += kv.second.bytes;
      slot.count += kv.second.count;
      out_base_[s] += kv.second.count;
      auto &pt = pred_[t];
      Agg moved = pt[l];
      pt.erase(l);
      Agg &r = pt[s];
      r.bytes += moved.bytes;
      r.count += moved.count;
    }
    for (const auto &kv : pred_[l]) {
      const int t = kv.first;
      Agg &slot = pred_[s][t];
      slot.bytes += kv.second.bytes;
      slot.count += kv.second.count;
      in_base_[s] += kv.second.count;
      auto &st = succ_[t];
      Agg moved = st[l];
      st.erase(l);
      Agg &r = st[s];
      r.bytes += moved.bytes;
      r.count += moved.count;
    }
    succ_[l].clear();
    pred_[l].clear();
    parent_[l] = s;
    if (track_) {
      // the merged root sits at the higher level; successors that fall at or
      // below it are raised, transitively (merges here never close a cycle)
      lvl_[s] = std::max(lvl_[s], lvl_[l]);
      std::vector<int> work{s};
      while (!work.empty()) {
        const int u = work.back();
        work.pop_back();
        for (const auto &kv : succ_[u])
          if (lvl_[kv.first] <= lvl_[u]) {
            lvl_[kv.first] = lvl_[u] + 1;
            work.push_back(kv.first);
          }
      }
    }
    return s;
  }

  struct Ref {
    int sk, dk, sr, dr;
  };
  // live edges sorted by (min member of src, min member of dst)
  std::vector<Ref> snapshot() {
    std::vector<Ref> out;
    for (int g = 0; g < static_cast<int>(parent_.size()); ++g) {
      if (find(g) != g) continue;
      for (const auto &kv : succ_[g]) out.push_back({minm_[g], minm_[kv.first], g, kv.first});
    }
    std::sort(out.begin(), out.end(), [](const Ref &a, const Ref &b) {
      return a.sk != b.sk ? a.sk < b.sk : a.dk < b.dk;
    });
    return out;
  }

  // a path a ~> b among live roots other than the direct edge a -> b
  bool path_besides_edge(int a, int b) {
    a = find(a);
    b = find(b);
    // with levels, only roots strictly below lvl(b) can lie on a path to b
    const int cut = track_ ? lvl_[b] : INT32_MAX;
    if (track_ && lvl_[a] >= cut) return false;
    auto wanted = [&](int t) { return t == b || !track_ || lvl_[t] < cut; };
    ++epoch_;
    std::vector<int> stack;
    stamp_[a] = epoch_;
    for (const auto &kv : succ_[a]) {
      if (kv.first == b) continue;
      if (stamp_[kv.first] != epoch_ && wanted(kv.first)) {
        stamp_[kv.first] = epoch_;
        stack.push_back(kv.first);
      }
    }
    while (!stack.empty()) {
      int u = stack.back();
      stack.pop_back();
      if (u == b) return true;
      for (const auto &kv : succ_[u])
        if (stamp_[kv.first] != epoch_ && wanted(kv.first)) {
          stamp_[kv.first] = epoch_;
          stack.push_back(kv.first);
        }
    }
    return false;
  }

  // canonical GroupedGraph: roots renumbered by ascending smallest member
  Meta build() {
    const int n = static_cast<int>(parent_.size());
    std::vector<int> roots;
    for (int g = 0; g < n; ++g)
      if (find(g) == g) roots.push_back(g);
    std::sort(roots.begin(), roots.end(), [&](int a, int b) { return minm_[a] < minm_[b]; });
    std::vector<int> idx(n, -1);
    for (size_t i = 0; i < roots.size(); ++i) idx[roots[i]] = static_cast<int>(i);
    Meta m;
    const size_t R = roots.size();
    m.members.resize(R);
    m.k.assign(R, 0);
    m.temp.assign(R, 0);
    m.perm.assign(R, 0);
    m.out.assign(R, 0);
    for (int g = 0; g < n; ++g) {
      int r = idx[find(g)];
      m.members[r].insert(m.members[r].end(), in_.members[g].begin(), in_.members[g].end());
      m.k[r] += in_.k[g];
      m.temp[r] = std::max(m.temp[r], in_.temp[g]);
      m.perm[r] += in_.perm[g];
      m.out[r] += in_.out[g];
    }
    for (auto &mm : m.members) std::sort(mm.begin(), mm.end());
    struct E4 {
      int s, d;
      int64_t b;
      int c;
    };
    std::vector<E4> es;
    for (int r : roots)
      for (const auto &kv : succ_[r]) es.push_back({idx[r], idx[kv.first], kv.second.bytes, kv.second.count});
    std::sort(es.begin(), es.end(), [](const E4 &a, const E4 &b) { return a.s != b.s ? a.s < b.s : a.d < b.d; });
    for (const E4 &e : es) {
      m.esrc.push_back(e.s);
      m.edst.push_back(e.d);
      m.ebytes.push_back(e.b);
      m.ecount.push_back(e.c);
    }
    m.group_of.resize(in_.group_of.size());
    for (size_t b = 0; b < in_.group_of.size(); ++b) m.group_of[b] = idx[find(in_.group_of[b])];
    return m;
  }

 private:
  const Meta &in_;
  bool track_;
  std::vector<int> parent_, minm_, out_base_, in_base_, stamp_, lvl_;
  int epoch_ = 0;
  std::vector<std::map<int, Agg>> succ_, pred_;
};

// meta_topo_order's acyclicity check + CycleError text (transforms.cpp:446-479)
void check_meta_acyclic(const Meta &m, const Base &b, const std::string &prefix) {
  const int V = m.V();
  std::vector<int> indeg(V, 0), off(V + 1, 0);
  for (size_t e = 0; e < m.esrc.size(); ++e) {
    indeg[m.edst[e]]++;
    off[m.esrc[e] + 1]++;
  }
  for (int v = 0; v < V; ++v) off[v + 1] += off[v];
  std::vector<int> q;
  for (int v = 0; v < V; ++v)
    if (!indeg[v]) q.push_back(v);
  size_t h = 0;
  while (h < q.size()) {
    int u = q[h++];
    for (int e = off[u]; e < off[u + 1]; ++e)
      if (--indeg[m.edst[e]] == 0) q.push_back(m.edst[e]);
  }
  if (static_cast<int>(q.size()) == V) return;
  std::string msg = prefix + "meta graph is cyclic; groups of base node ids {";
  bool first = true;
  for (int v = 0; v < V; ++v)
    if (indeg[v] > 0) {
      msg += (first ? "" : ", ") + std::to_string(b.id[m.members[v].front()]);
      first = false;
    }
  throw VErr(msg + "} remain");
}

Meta apply_colocation(const Meta &gg, const Base &b) {
  Merger mg(gg);
  std::unordered_map<int32_t, int> first_group;
  for (int i = 0; i < b.n; ++i) {
    if (b.label[i] < 0) continue;
    auto ins = first_group.emplace(b.label[i], gg.group_of[i]);
    if (!ins.second) mg.unite(ins.first->second, gg.group_of[i]);
  }
  Meta out = mg.build();
  check_meta_acyclic(out, b, "colocation-induced cycle: ");
  return out;
}

Meta apply_coplacement(const Meta &gg, const Base &b) {
  Merger mg(gg, true);
  for (int i = 0; i < b.n; ++i) {
    if (!b.has_pair[i]) continue;
    int peer = b.index_of(b.pair[i]);
    if (peer < i) continue;  // each pair once, ascending
    int x = mg.find(gg.group_of[i]), y = mg.find(gg.group_of[peer]);
    if (x == y) continue;
    if (mg.path_besides_edge(x, y) || mg.path_besides_edge(y, x)) continue;  // would close a cycle
    mg.unite(x, y);
  }
  bool changed = true;
  while (changed) {
    changed = false;
    for (const auto &r : mg.snapshot()) {
      int x = mg.find(r.sr), y = mg.find(r.dr);
      if (x == y) continue;
      if (mg.out_base(x) == 1) {
        mg.unite(x, y);
        changed = true;
      }
    }
  }
  return mg.build();
}

Meta fuse_operators(const Meta &gg, const Base &b) {
  Merger mg(gg, true);
  // affinity classes over base nodes: colocation label or coplace pair
  std::vector<int> par(b.n);
  std::iota(par.begin(), par.end(), 0);
  auto f = [&](int x) {
    while (par[x] != x) {
      par[x] = par[par[x]];
      x = par[x];
    }
    return x;
  };
  auto un = [&](int x, int y) {
    x = f(x);
    y = f(y);
    if (x != y) par[std::max(x, y)] = std::min(x, y);
  };
  std::unordered_map<int32_t, int> first_label;
  for (int i = 0; i < b.n; ++i) {
    if (b.label[i] >= 0) {
      auto ins = first_label.emplace(b.label[i], i);
      if (!ins.second) un(ins.first->second, i);
    }
    if (b.has_pair[i]) un(i, b.index_of(b.pair[i]));
  }
  std::vector<int> aff(b.n), asize(b.n, 0);
  for (int i = 0; i < b.n; ++i) asize[aff[i] = f(i)]++;
  std::vector<std::vector<int>> sets(gg.V());  // sorted, unique affinity roots
  for (int i = 0; i < b.n; ++i)
    if (asize[aff[i]] >= 2) sets[mg.find(gg.group_of[i])].push_back(aff[i]);
  for (auto &st : sets) {
    std::sort(st.begin(), st.end());
    st.erase(std::unique(st.begin(), st.end()), st.end());
  }
  auto affine = [&](int x, int y) {
    const auto &a = sets[x], &c = sets[y];
    size_t i = 0, j = 0;
    while (i < a.size() && j < c.size()) {
      if (a[i] == c[j]) return true;
      if (a[i] < c[j]) ++i;
      else ++j;
    }
    return false;
  };
  bool changed = true;
  while (changed) {
    changed = false;
    for (const auto &r : mg.snapshot()) {
      int x = mg.find(r.sr), y = mg.find(r.dr);
      if (x == y || !affine(x, y)) continue;
      if (mg.out_base(x) != 1 && mg.in_base(y) != 1) continue;
      int sv = mg.unite(x, y);
      int ls = sv == x ? y : x;
      std::vector<int> merged;
      std::set_union(sets[sv].begin(), sets[sv].end(), sets[ls].begin(), sets[ls].end(),
                     std::back_inserter(merged));
      sets[sv].swap(merged);
      sets[ls].clear();
      changed = true;
    }
  }
  return mg.build();
}

void put(char *msg, int len, const std::string &s) {
  if (msg && len > 0) std::snprintf(msg, static_cast<size_t>(len), "%s", s.c_str());
}

}  // namespace

struct bx_grouped {
  Base base;
  Meta meta;
  std::vector<int32_t> in_off, in_edge, out_off, members, member_off;
  std::vector<int64_t> first_id;
};

extern "C" {

int bx_grouped_create(const bx_base_graph *in, int32_t pipeline, bx_grouped **out, char *msg, int msglen) {
  *out = nullptr;
  try {
    auto G = new bx_grouped();
    G->base = make_graph(*in);
    Meta m = singleton_groups(G->base);
    if (pipeline >= 0) {  // build_grouped (bench.cpp:43-49)
      m = apply_colocation(m, G->base);
      if (pipeline & BX_PIPE_COPLACEMENT) m = apply_coplacement(m, G->base);
      if (pipeline & BX_PIPE_FUSION) m = fuse_operators(m, G->base);
    }
    G->meta = std::move(m);
    const Meta &M = G->meta;
    const int V = M.V(), E = static_cast<int>(M.esrc.size());
    G->in_off.assign(V + 1, 0);
    G->out_off.assign(V + 1, 0);
    G->in_edge.assign(std::max(E, 1), 0);
    char emsg[256];
    bx_build_adjacency(V, E, M.esrc.data(), M.edst.data(), G->in_off.data(), G->in_edge.data(),
                       G->out_off.data(), emsg, sizeof emsg);
    G->member_off.push_back(0);
    for (int v = 0; v < V; ++v) {
      for (int b : M.members[v]) G->members.push_back(b);
      G->member_off.push_back(static_cast<int32_t>(G->members.size()));
      G->first_id.push_back(G->base.id[M.members[v].front()]);
    }
    *out = G;
    put(msg, msglen, "");
    return BX_OK;
  } catch (const VErr &e) {
    put(msg, msglen, e.what());
    return BX_VALIDATION;
  } catch (const std::exception &e) {
    put(msg, msglen, std::string("ingest failure: ") + e.what());
    return BX_RUNTIME;
  }
}

int bx_grouped_view(const bx_grouped *G, bx_graph *meta, bx_grouping *grouping) {
  const Meta &M = G->meta;
  meta->V = M.V();
  meta->E = static_cast<int32_t>(M.esrc.size());
  meta->compute_us = M.k.data();
  meta->temp_bytes = M.temp.data();
  meta->perm_bytes = M.perm.data();
  meta->out_bytes = M.out.data();
  meta->esrc = M.esrc.data();
  meta->edst = M.edst.data();
  meta->tensor_bytes = M.ebytes.data();
  meta->in_off = G->in_off.data();
  meta->in_edge = G->in_edge.data();
  meta->out_off = G->out_off.data();
  meta->first_id = G->first_id.data();
  if (grouping) {
    grouping->base_nodes = G->base.n;
    grouping->base_ids = G->base.id.data();
    grouping->group_of = M.group_of.data();
    grouping->members = G->members.data();
    grouping->member_off = G->member_off.data();
    grouping->edge_base_count = M.ecount.data();
  }
  return BX_OK;
}

void bx_grouped_destroy(bx_grouped *G) { delete G; }

}  // extern "C"

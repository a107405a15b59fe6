// TEST INFRASTRUCTURE ONLY — the parity checker, never the product.
//
// A flat C ABI over the UNMODIFIED reference `dagsched` sources
// (/root/reference/proj/src/{graph,transforms,cost_model,placers,simulator,
// generator}.cpp, compiled in place by oracle/Makefile into oracle/_ref/).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference legs load the resulting libdagsched_ref.so.
//
// Every entry point forwards to the reference's own public API:
//   make_graph              proj/src/graph.cpp:99
//   apply_colocation        proj/src/transforms.cpp:329
//   apply_coplacement       proj/src/transforms.cpp:353
//   fuse_operators          proj/src/transforms.cpp:390
//   meta_topo_order         proj/src/transforms.cpp:446
//   comm_time               proj/src/cost_model.cpp:30
//   place_mtopo/metf/msct   proj/src/placers.cpp:299-365
//   schedulable_time        proj/src/placers.cpp:83
//   simulate                proj/src/simulator.cpp:273
//   critical_path_us        proj/src/simulator.cpp:296
//   trace_to_csv            proj/src/simulator.cpp:311
//   parse_graph/graph_to_json         proj/src/graph.cpp:196-309
//   parse/save_comm_model             proj/src/cost_model.cpp:71-134
//   placement_to_json/_from_json      proj/src/placers.cpp:367-432
//   generate_graph          proj/src/generator.cpp:173
// The pipeline composition mirrors build_grouped (proj/src/bench.cpp:43-49)
// and the sweep's capacity rule bench_capacity (proj/src/bench.cpp:77-87);
// bench.cpp itself is not linked because it needs the Eigen-based LP.
// The LP (proj/src/lp.cpp) needs Eigen3, absent from this image, so
// round_and_extract is restated in oracle/restate.c instead.

#include <omp.h>

#include <chrono>
#include <cstdio>
#include <fstream>
#include <sstream>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <optional>
#include <string>
#include <vector>

#include "dagsched/cost_model.hpp"
#include "dagsched/errors.hpp"
#include "dagsched/generator.hpp"
#include "dagsched/graph.hpp"
#include "dagsched/lp.hpp"
#include "dagsched/oracle.hpp"
#include "dagsched/placers.hpp"
#include "dagsched/simulator.hpp"
#include "dagsched/transforms.hpp"

using namespace dagsched;

namespace {

struct RefGraph {
  std::shared_ptr<const ProfiledGraph> base;
  GroupedGraph gg;
};

int kind_code(const Error& e) {
  switch (e.kind()) {
    case ErrorKind::Validation: return 2;
    case ErrorKind::Infeasible: return 3;
    case ErrorKind::Solver: return 4;
  }
  return 9;
}

void put(char* err, int errlen, const std::string& s) {
  if (!err || errlen <= 0) return;
  std::snprintf(err, static_cast<size_t>(errlen), "%s", s.c_str());
}

template <typename F>
int guarded(char* err, int errlen, F&& f) {
  try {
    f();
    put(err, errlen, "");
    return 0;
  } catch (const Error& e) {
    put(err, errlen, e.what());
    return kind_code(e);
  } catch (const std::exception& e) {
    put(err, errlen, std::string("std::exception: ") + e.what());
    return 9;
  }
}

CommModel make_cm(double intercept, double per_byte, int mode) {
  return CommModel{intercept, per_byte,
                   mode == 1 ? CommMode::Parallel : CommMode::Sequential};
}

DeviceRoster make_roster(int n, const int64_t* caps) {
  DeviceRoster r;
  for (int i = 0; i < n; ++i) r.devices.push_back({i, caps[i]});
  return r;
}

void export_placement(const Placement& p, int32_t* device_of, int64_t* start,
                      int32_t* exec_order, int32_t* exec_off) {
  int V = static_cast<int>(p.device_of.size());
  for (int j = 0; j < V; ++j) {
    device_of[j] = p.device_of[j];
    start[j] = p.start_us[j];
  }
  int pos = 0;
  exec_off[0] = 0;
  for (size_t d = 0; d < p.exec_order.size(); ++d) {
    for (int j : p.exec_order[d]) exec_order[pos++] = j;
    exec_off[d + 1] = pos;
  }
}

Placement import_placement(const GroupedGraph& gg, int n,
                           const int32_t* device_of, const int32_t* exec_order,
                           const int32_t* exec_off) {
  Placement p;
  p.algorithm = "external";
  p.device_of.assign(device_of, device_of + gg.node_count());
  p.start_us.assign(gg.node_count(), 0);
  p.exec_order.assign(n, {});
  for (int d = 0; d < n; ++d) {
    for (int i = exec_off[d]; i < exec_off[d + 1]; ++i) {
      p.exec_order[d].push_back(exec_order[i]);
    }
  }
  return p;
}

}  // namespace

extern "C" {

// Builds the reference ProfiledGraph (make_graph) and GroupedGraph.
// pipeline: -1 = singleton_groups only; otherwise bit0 ignored (colocation
// always runs, as in build_grouped), bit1 = co-placement, bit2 = fusion.
// coloc_label[i] < 0 means no colocation_group, else the label "g<k>";
// has_pair[i] != 0 means coplace_pair = pair_id[i].
int ref_graph_new(int32_t nn, const int64_t* id, const int64_t* k,
                  const int64_t* temp, const int64_t* perm, const int64_t* out,
                  const int32_t* coloc_label, const uint8_t* has_pair,
                  const int64_t* pair_id, int32_t ne, const int64_t* src,
                  const int64_t* dst, const int64_t* bytes, int32_t pipeline,
                  void** handle, char* err, int errlen) {
  *handle = nullptr;
  return guarded(err, errlen, [&] {
    std::vector<OpNode> nodes(nn);
    for (int i = 0; i < nn; ++i) {
      OpNode& n = nodes[i];
      n.id = id[i];
      n.name = "n" + std::to_string(id[i]);
      n.compute_time_us = k[i];
      n.temp_mem_bytes = temp[i];
      n.perm_mem_bytes = perm[i];
      n.out_mem_bytes = out[i];
      if (coloc_label && coloc_label[i] >= 0) {
        n.colocation_group = "g" + std::to_string(coloc_label[i]);
      }
      if (has_pair && has_pair[i]) n.coplace_pair = pair_id[i];
    }
    std::vector<Edge> edges(ne);
    for (int e = 0; e < ne; ++e) edges[e] = {src[e], dst[e], bytes[e]};
    auto rg = std::make_unique<RefGraph>();
    rg->base = std::make_shared<ProfiledGraph>(
        make_graph(std::move(nodes), std::move(edges)));
    if (pipeline < 0) {
      rg->gg = singleton_groups(rg->base);
    } else {
      rg->gg = apply_colocation(rg->base);
      if (pipeline & 2) rg->gg = apply_coplacement(rg->gg);
      if (pipeline & 4) rg->gg = fuse_operators(rg->gg);
    }
    *handle = rg.release();
  });
}

void ref_graph_free(void* h) { delete static_cast<RefGraph*>(h); }

void ref_graph_sizes(void* h, int32_t* base_v, int32_t* base_e, int32_t* V,
                     int32_t* E, int32_t* members_total) {
  auto* rg = static_cast<RefGraph*>(h);
  *base_v = rg->base->node_count();
  *base_e = rg->base->edge_count();
  *V = rg->gg.node_count();
  *E = rg->gg.edge_count();
  int m = 0;
  for (const MetaNode& n : rg->gg.nodes) m += static_cast<int>(n.members.size());
  *members_total = m;
}

// Meta graph export: aggregates per meta node, meta edges in (src, dst)
// order, group_of per base index, members flattened with offsets.
void ref_graph_meta(void* h, int64_t* k, int64_t* temp, int64_t* perm,
                    int64_t* out, int32_t* esrc, int32_t* edst, int64_t* ebytes,
                    int32_t* ecount, int32_t* group_of, int32_t* members,
                    int32_t* member_off) {
  auto* rg = static_cast<RefGraph*>(h);
  const GroupedGraph& gg = rg->gg;
  int pos = 0;
  member_off[0] = 0;
  for (int i = 0; i < gg.node_count(); ++i) {
    const MetaNode& m = gg.nodes[i];
    k[i] = m.compute_time_us;
    temp[i] = m.temp_mem_bytes;
    perm[i] = m.perm_mem_bytes;
    out[i] = m.out_mem_bytes;
    for (int b : m.members) members[pos++] = b;
    member_off[i + 1] = pos;
  }
  for (int e = 0; e < gg.edge_count(); ++e) {
    esrc[e] = gg.edges[e].src;
    edst[e] = gg.edges[e].dst;
    ebytes[e] = gg.edges[e].tensor_bytes;
    ecount[e] = gg.edges[e].base_count;
  }
  for (size_t b = 0; b < gg.group_of.size(); ++b) group_of[b] = gg.group_of[b];
}

// Base graph export after make_graph's canonical sort (nodes by id, edges by
// (src index, dst index)); edge endpoints as dense indices.
void ref_graph_base(void* h, int64_t* id, int32_t* esrc, int32_t* edst,
                    int64_t* ebytes) {
  auto* rg = static_cast<RefGraph*>(h);
  const ProfiledGraph& g = *rg->base;
  for (int i = 0; i < g.node_count(); ++i) id[i] = g.nodes[i].id;
  for (int e = 0; e < g.edge_count(); ++e) {
    esrc[e] = g.index_of(g.edges[e].src);
    edst[e] = g.index_of(g.edges[e].dst);
    ebytes[e] = g.edges[e].tensor_bytes;
  }
}

int ref_meta_topo_order(void* h, int32_t* order, char* err, int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    std::vector<int> o = meta_topo_order(rg->gg);
    for (size_t i = 0; i < o.size(); ++i) order[i] = o[i];
  });
}

int64_t ref_critical_path(void* h) {
  return critical_path_us(static_cast<RefGraph*>(h)->gg);
}

int ref_comm_time(double intercept, double per_byte, int64_t bytes,
                  int64_t* out, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    *out = comm_time(make_cm(intercept, per_byte, 0), bytes);
  });
}

int64_t ref_max_comm_time(void* h, double intercept, double per_byte) {
  return max_comm_time(static_cast<RefGraph*>(h)->gg,
                       make_cm(intercept, per_byte, 0));
}

// Ceil(factor * (total reserve / n + max reserve)), proj/src/bench.cpp:77-87.
int64_t ref_bench_capacity(void* h, int32_t n, double factor) {
  const GroupedGraph& gg = static_cast<RefGraph*>(h)->gg;
  bytes_t total = 0, largest = 0;
  for (const MetaNode& m : gg.nodes) {
    total += reserve_bytes(m);
    largest = std::max(largest, reserve_bytes(m));
  }
  double need = static_cast<double>(total) / n + static_cast<double>(largest);
  return static_cast<bytes_t>(std::ceil(need * factor));
}

// algo: 0 m-topo, 1 m-etf, 2 m-sct (fav_child may be NULL: empty map).
// stats3: discarded, excluded, awake. wall_ns: the placer call alone
// (run_placer's scope, proj/src/bench.cpp:55-74, minus the LP).
int ref_place(void* h, int32_t algo, int32_t n, const int64_t* caps,
              double intercept, double per_byte, int32_t mode,
              const int32_t* fav_child, int32_t* device_of, int64_t* start,
              int32_t* exec_order, int32_t* exec_off, int64_t* stats3,
              int64_t* wall_ns, char* err, int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    DeviceRoster roster = make_roster(n, caps);
    CommModel cm = make_cm(intercept, per_byte, mode);
    PlacerStats stats;
    Placement p;
    FavoriteMap fav;
    if (algo == 2 && fav_child) {
      fav.fav_child.assign(fav_child, fav_child + rg->gg.node_count());
      fav.fav_parent.assign(rg->gg.node_count(), -1);
      for (int i = 0; i < rg->gg.node_count(); ++i) {
        if (fav_child[i] >= 0 && fav_child[i] < rg->gg.node_count()) {
          fav.fav_parent[fav_child[i]] = i;
        }
      }
    }
    auto t0 = std::chrono::steady_clock::now();
    if (algo == 0) {
      p = place_mtopo(rg->gg, roster, cm);
    } else if (algo == 1) {
      p = place_metf(rg->gg, roster, cm, &stats);
    } else {
      p = place_msct(rg->gg, roster, cm, fav, &stats);
    }
    auto t1 = std::chrono::steady_clock::now();
    if (wall_ns) {
      *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0)
                     .count();
    }
    export_placement(p, device_of, start, exec_order, exec_off);
    if (stats3) {
      stats3[0] = stats.discarded_pairs;
      stats3[1] = stats.excluded_devices;
      stats3[2] = stats.awake_reservations;
    }
  });
}

// Times `reps` back-to-back placer calls on one graph; returns per-call ns.
int ref_place_timed(void* h, int32_t algo, int32_t n, const int64_t* caps,
                    double intercept, double per_byte, int32_t mode,
                    const int32_t* fav_child, int32_t reps, int64_t* ns_each,
                    char* err, int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    DeviceRoster roster = make_roster(n, caps);
    CommModel cm = make_cm(intercept, per_byte, mode);
    FavoriteMap fav;
    if (algo == 2 && fav_child) {
      fav.fav_child.assign(fav_child, fav_child + rg->gg.node_count());
      fav.fav_parent.assign(rg->gg.node_count(), -1);
    }
    for (int r = 0; r < reps; ++r) {
      PlacerStats stats;
      auto t0 = std::chrono::steady_clock::now();
      Placement p = algo == 0   ? place_mtopo(rg->gg, roster, cm)
                    : algo == 1 ? place_metf(rg->gg, roster, cm, &stats)
                                : place_msct(rg->gg, roster, cm, fav, &stats);
      auto t1 = std::chrono::steady_clock::now();
      ns_each[r] = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0)
                       .count();
      (void)p;
    }
  });
}

// Batched placement of many (graph, roster) problems with the reference's
// own sweep pattern: #pragma omp parallel for schedule(dynamic)
// (proj/src/bench.cpp:121). Returns wall ns of the whole batch; statuses
// per problem (0 ok / error kind) and makespan-free checksum per problem
// (sum of start_us + device_of) so the GPU batch can be cross-checked.
int ref_place_batch(int32_t count, void* const* graphs, const int32_t* algo,
                    const int32_t* n, const int64_t* caps /* count x maxn */,
                    int32_t maxn, double intercept, double per_byte,
                    int32_t mode, int32_t threads, int32_t* status,
                    int64_t* checksum, int64_t* wall_ns) {
  if (threads > 0) omp_set_num_threads(threads);
  auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < count; ++i) {
    auto* rg = static_cast<RefGraph*>(graphs[i]);
    try {
      DeviceRoster roster = make_roster(n[i], caps + static_cast<size_t>(i) * maxn);
      CommModel cm = make_cm(intercept, per_byte, mode);
      PlacerStats stats;
      Placement p = algo[i] == 0 ? place_mtopo(rg->gg, roster, cm)
                                 : place_metf(rg->gg, roster, cm, &stats);
      int64_t sum = 0;
      for (size_t j = 0; j < p.device_of.size(); ++j) {
        sum += p.start_us[j] * 131 + p.device_of[j];
      }
      checksum[i] = sum;
      status[i] = 0;
    } catch (const Error& e) {
      status[i] = kind_code(e);
      checksum[i] = 0;
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  *wall_ns =
      std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  return 0;
}

// schedulable_time (proj/src/placers.cpp:83) against an explicit state.
int ref_schedulable_time(void* h, int32_t n, int32_t mode, double intercept,
                         double per_byte, const int64_t* dev_free,
                         const int64_t* xfer_tail, const int32_t* device_of,
                         const int64_t* finish, const int64_t* cache,
                         int32_t j, int32_t p, int64_t* out, char* err,
                         int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    int V = rg->gg.node_count();
    PlacerState st(V, n, mode == 1 ? CommMode::Parallel : CommMode::Sequential);
    st.dev_free.assign(dev_free, dev_free + n);
    st.xfer_tail.assign(xfer_tail, xfer_tail + n);
    st.device_of.assign(device_of, device_of + V);
    st.finish_us.assign(finish, finish + V);
    st.cache_arrival.assign(cache, cache + static_cast<size_t>(V) * n);
    *out = schedulable_time(st, j, p, rg->gg, make_cm(intercept, per_byte, mode));
  });
}

// simulate (proj/src/simulator.cpp:273). mem_mode: 0 GraphStatic,
// 1 TrainingPersistent. dev3n: peak, busy, idle per device.
// xfer4: transfer_count, transfer_bytes, duplicate_transfers, cache_hits.
int ref_simulate(void* h, int32_t n, const int64_t* caps, double intercept,
                 double per_byte, int32_t mode, int32_t mem_mode,
                 const int32_t* device_of, const int32_t* exec_order,
                 const int32_t* exec_off, int64_t* makespan, int64_t* start,
                 int64_t* dev3n, int64_t* xfer4, int64_t* wall_ns, char* err,
                 int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    DeviceRoster roster = make_roster(n, caps);
    CommModel cm = make_cm(intercept, per_byte, mode);
    Placement p = import_placement(rg->gg, n, device_of, exec_order, exec_off);
    auto t0 = std::chrono::steady_clock::now();
    SimReport r = simulate(rg->gg, p, roster, cm,
                           mem_mode == 1 ? MemoryMode::TrainingPersistent
                                         : MemoryMode::GraphStatic);
    auto t1 = std::chrono::steady_clock::now();
    if (wall_ns) {
      *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0)
                     .count();
    }
    *makespan = r.makespan_us;
    for (int j = 0; j < rg->gg.node_count(); ++j) start[j] = r.start_us[j];
    for (int d = 0; d < n; ++d) {
      dev3n[3 * d + 0] = r.devices[d].peak_bytes;
      dev3n[3 * d + 1] = r.devices[d].busy_us;
      dev3n[3 * d + 2] = r.devices[d].idle_us;
    }
    xfer4[0] = r.transfer_count;
    xfer4[1] = r.transfer_bytes;
    xfer4[2] = r.duplicate_transfers;
    xfer4[3] = r.cache_hits;
  });
}

// generate_graph (proj/src/generator.cpp:173). family: 0 branchy,
// 1 layered-chain, 2 random-dag. Two-phase: call with cap_nodes/cap_edges
// too small (e.g. 0) to learn the sizes, then again with buffers.
int ref_generate(int32_t family, int32_t node_count, int32_t branching,
                 int32_t layers, double edge_prob, uint64_t seed,
                 const int64_t* ranges /* 10: compute,tensor,temp,perm,out */,
                 double colocate_edge_frac, double coplace_frac,
                 int32_t cap_nodes, int32_t cap_edges, int32_t* nn,
                 int32_t* ne, int64_t* id, int64_t* k, int64_t* temp,
                 int64_t* perm, int64_t* out, int32_t* coloc_label,
                 uint8_t* has_pair, int64_t* pair_id, int64_t* src,
                 int64_t* dst, int64_t* bytes, char* err, int errlen) {
  return guarded(err, errlen, [&] {
    GenSpec spec;
    spec.family = family == 0   ? GraphFamily::Branchy
                  : family == 1 ? GraphFamily::LayeredChain
                                : GraphFamily::RandomDag;
    spec.node_count = node_count;
    spec.branching = branching;
    spec.layers = layers;
    spec.edge_prob = edge_prob;
    spec.seed = seed;
    if (ranges) {
      spec.compute_min_us = ranges[0];
      spec.compute_max_us = ranges[1];
      spec.tensor_min_bytes = ranges[2];
      spec.tensor_max_bytes = ranges[3];
      spec.temp_min_bytes = ranges[4];
      spec.temp_max_bytes = ranges[5];
      spec.perm_min_bytes = ranges[6];
      spec.perm_max_bytes = ranges[7];
      spec.out_min_bytes = ranges[8];
      spec.out_max_bytes = ranges[9];
    }
    spec.colocate_edge_frac = colocate_edge_frac;
    spec.coplace_frac = coplace_frac;
    ProfiledGraph g = generate_graph(spec);
    *nn = g.node_count();
    *ne = g.edge_count();
    if (cap_nodes < g.node_count() || cap_edges < g.edge_count()) return;
    for (int i = 0; i < g.node_count(); ++i) {
      const OpNode& n = g.nodes[i];
      id[i] = n.id;
      k[i] = n.compute_time_us;
      temp[i] = n.temp_mem_bytes;
      perm[i] = n.perm_mem_bytes;
      out[i] = n.out_mem_bytes;
      coloc_label[i] = n.colocation_group
                           ? std::stoi(n.colocation_group->substr(1))
                           : -1;
      has_pair[i] = n.coplace_pair ? 1 : 0;
      pair_id[i] = n.coplace_pair ? *n.coplace_pair : 0;
    }
    for (int e = 0; e < g.edge_count(); ++e) {
      src[e] = g.edges[e].src;
      dst[e] = g.edges[e].dst;
      bytes[e] = g.edges[e].tensor_bytes;
    }
  });
}

// Copies a string result into a caller buffer (two-phase: needed first).
static int put_text(const std::string& s, char* buf, int64_t buflen, int64_t* needed) {
  *needed = static_cast<int64_t>(s.size()) + 1;
  if (!buf || buflen < *needed) return 1;
  std::memcpy(buf, s.data(), s.size());
  buf[s.size()] = '\0';
  return 0;
}

// simulate with SimOptions{record_trace = true}, then trace_to_csv.
int ref_simulate_trace_csv(void* h, int32_t n, const int64_t* caps, double intercept, double per_byte, int32_t mode,
                           int32_t mem_mode, const int32_t* device_of, const int32_t* exec_order,
                           const int32_t* exec_off, char* buf, int64_t buflen, int64_t* needed, int64_t* events,
                           char* err, int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  *needed = 0;
  return guarded(err, errlen, [&] {
    SimOptions opt;
    opt.record_trace = true;
    Placement p = import_placement(rg->gg, n, device_of, exec_order, exec_off);
    SimReport r = simulate(rg->gg, p, make_roster(n, caps), make_cm(intercept, per_byte, mode),
                           mem_mode == 1 ? MemoryMode::TrainingPersistent : MemoryMode::GraphStatic, opt);
    *events = static_cast<int64_t>(r.trace.size());
    put_text(trace_to_csv(r.trace), buf, buflen, needed);
  });
}

// parse_graph(text) then graph_to_json of the result.
int ref_graph_json_roundtrip(const char* text, int64_t len, char* buf, int64_t buflen, int64_t* needed, char* err,
                             int errlen) {
  *needed = 0;
  return guarded(err, errlen, [&] {
    ProfiledGraph g = parse_graph(std::string(text, static_cast<size_t>(len)));
    put_text(graph_to_json(g), buf, buflen, needed);
  });
}

// graph_to_json of a handle's base graph (names "n<id>", groups "g<label>").
int ref_graph_to_json(void* h, char* buf, int64_t buflen, int64_t* needed) {
  return put_text(graph_to_json(*static_cast<RefGraph*>(h)->base), buf, buflen, needed);
}

// parse_comm_model(text) then save_comm_model's text (written to a temp file
// by the reference and read back).
int ref_comm_model_roundtrip(const char* text, int64_t len, double* ic, double* pb, int32_t* mode, char* buf,
                             int64_t buflen, int64_t* needed, char* err, int errlen) {
  *needed = 0;
  return guarded(err, errlen, [&] {
    CommModel cm = parse_comm_model(std::string(text, static_cast<size_t>(len)));
    *ic = cm.intercept_us;
    *pb = cm.us_per_byte;
    *mode = cm.mode == CommMode::Parallel ? 1 : 0;
    char path[] = "/tmp/bx_cm_XXXXXX";
    int fd = mkstemp(path);
    if (fd >= 0) close(fd);
    save_comm_model(cm, path);
    std::ifstream in(path);
    std::ostringstream b;
    b << in.rdbuf();
    std::remove(path);
    put_text(b.str(), buf, buflen, needed);
  });
}

// placement_to_json of an external placement with a simulated report.
int ref_placement_to_json(void* h, const char* algorithm, int32_t n, const int32_t* device_of,
                          const int32_t* exec_order, const int32_t* exec_off, const int64_t* sim_start,
                          int64_t makespan, const int64_t* peaks, char* buf, int64_t buflen, int64_t* needed) {
  auto* rg = static_cast<RefGraph*>(h);
  Placement p = import_placement(rg->gg, n, device_of, exec_order, exec_off);
  p.algorithm = algorithm;
  std::vector<micros_t> st(sim_start, sim_start + rg->gg.node_count());
  std::vector<bytes_t> pk(peaks, peaks + n);
  return put_text(placement_to_json(rg->gg, p, st, makespan, pk), buf, buflen, needed);
}

int ref_placement_from_json(void* h, const char* text, int64_t len, int32_t n, char* algorithm, int algolen,
                            int32_t* device_of, int64_t* start, int32_t* exec_order, int32_t* exec_off, char* err,
                            int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    Placement p = placement_from_json(rg->gg, std::string(text, static_cast<size_t>(len)), n);
    put(algorithm, algolen, p.algorithm);
    export_placement(p, device_of, start, exec_order, exec_off);
  });
}

// ref_place_batch with the full placements exported: problem i writes its
// device_of / start_us / exec_order at element offset voff[i] of the flat
// arrays, exec_off at eoff[i], stats at 3*i (the bench compares every one of
// the sweep's problems with the GPU, not a checksum).
int ref_place_batch_full(int32_t count, void* const* graphs, const int32_t* algo, const int32_t* n,
                         const int64_t* caps, int32_t maxn, double intercept, double per_byte, int32_t mode,
                         int32_t threads, const int64_t* voff, const int64_t* eoff, int32_t* device_of,
                         int64_t* start, int32_t* exec_order, int32_t* exec_off, int64_t* stats3, int32_t* status,
                         int64_t* wall_ns) {
  if (threads > 0) omp_set_num_threads(threads);
  auto t0 = std::chrono::steady_clock::now();
#pragma omp parallel for schedule(dynamic)
  for (int i = 0; i < count; ++i) {
    auto* rg = static_cast<RefGraph*>(graphs[i]);
    try {
      DeviceRoster roster = make_roster(n[i], caps + static_cast<size_t>(i) * maxn);
      CommModel cm = make_cm(intercept, per_byte, mode);
      PlacerStats st;
      Placement p = algo[i] == 0 ? place_mtopo(rg->gg, roster, cm) : place_metf(rg->gg, roster, cm, &st);
      export_placement(p, device_of + voff[i], start + voff[i], exec_order + voff[i], exec_off + eoff[i]);
      stats3[3 * i + 0] = st.discarded_pairs;
      stats3[3 * i + 1] = st.excluded_devices;
      stats3[3 * i + 2] = st.awake_reservations;
      status[i] = 0;
    } catch (const Error& e) {
      status[i] = kind_code(e);
    }
  }
  auto t1 = std::chrono::steady_clock::now();
  *wall_ns = std::chrono::duration_cast<std::chrono::nanoseconds>(t1 - t0).count();
  return 0;
}

// oracle_makespan (proj/src/oracle.cpp:185-212). capacity < 0: none.
int ref_oracle_makespan(void* h, int32_t n, double intercept, double per_byte, int32_t mode,
                        int64_t capacity, int32_t mem_mode, int32_t max_nodes, int32_t max_devices,
                        int64_t max_extensions, int64_t* out, char* err, int errlen) {
  auto* rg = static_cast<RefGraph*>(h);
  return guarded(err, errlen, [&] {
    OracleLimits lim;
    lim.max_nodes = max_nodes;
    lim.max_devices = max_devices;
    lim.max_extensions = max_extensions;
    std::optional<bytes_t> cap;
    if (capacity >= 0) cap = capacity;
    *out = oracle_makespan(rg->gg, n, make_cm(intercept, per_byte, mode), cap,
                           mem_mode == 1 ? MemoryMode::TrainingPersistent : MemoryMode::GraphStatic, lim);
  });
}

}  // extern "C"

// proj/src/placers_b200.cpp — the reference-side shim: the
// dagsched placer entry points (proj/include/dagsched/placers.hpp:73-89) with
// their reference signatures, forwarded to the B200 engine's C ABI
// (include/baechi_b200.h, bx_place). A maintainer builds it instead of the
// three place_* definitions of placers.cpp and links libbaechi_b200.so.
// Errors come back as the reference's exception types with its what() text.
#include <algorithm>
#include <stdexcept>
#include <vector>

#include "baechi_b200.h"
#include "dagsched/errors.hpp"
#include "dagsched/lp.hpp"
#include "dagsched/placers.hpp"

namespace dagsched {
namespace {
struct Flat {  // GroupedGraph -> bx_graph (arrays live as long as the call)
  std::vector<int64_t> k, temp, perm, out, bytes, first_id;
  std::vector<int32_t> src, dst, in_off, in_edge, out_off;
  bx_graph g{};
  explicit Flat(const GroupedGraph& gg) {
    const int V = gg.node_count(), E = gg.edge_count();
    for (const MetaNode& m : gg.nodes) {
      k.push_back(m.compute_time_us);
      temp.push_back(m.temp_mem_bytes);
      perm.push_back(m.perm_mem_bytes);
      out.push_back(m.out_mem_bytes);
      first_id.push_back(gg.base->nodes[m.members.front()].id);
    }
    for (const MetaEdge& e : gg.edges) {
      src.push_back(e.src);
      dst.push_back(e.dst);
      bytes.push_back(e.tensor_bytes);
    }
    in_off.assign(V + 1, 0);
    out_off.assign(V + 1, 0);
    in_edge.assign(std::max(E, 1), 0);
    char msg[256];
    bx_build_adjacency(V, E, src.data(), dst.data(), in_off.data(), in_edge.data(), out_off.data(), msg,
                       sizeof msg);  // == gg.in_edges / out_edges
    g = {V, E, k.data(), temp.data(), perm.data(), out.data(), src.data(), dst.data(), bytes.data(),
         in_off.data(), in_edge.data(), out_off.data(), first_id.data()};
  }
};

[[noreturn]] void rethrow(int status, const char* msg) {
  switch (status) {
    case BX_VALIDATION: throw ValidationError(msg);
    case BX_INFEASIBLE: throw InfeasibleError(msg);
    case BX_SOLVER: throw SolverError(msg);
    default: throw std::runtime_error(msg);  // BX_RUNTIME: CUDA failure
  }
}

Placement run(const GroupedGraph& gg, const DeviceRoster& r, const CommModel& cm, int algo,
              const FavoriteMap* fav, PlacerStats* stats, const char* name) {
  Flat f(gg);
  std::vector<int64_t> caps;
  for (const Device& d : r.devices) caps.push_back(d.capacity_bytes);
  bx_job job{0,
             algo,
             r.count(),
             caps.data(),
             {cm.intercept_us, cm.us_per_byte, cm.mode == CommMode::Parallel ? BX_COMM_PARALLEL : BX_COMM_SEQUENTIAL},
             fav && !fav->fav_child.empty() ? fav->fav_child.data() : nullptr,
             fav ? static_cast<int32_t>(fav->fav_child.size()) : 0};
  const int V = gg.node_count();
  std::vector<int32_t> dev(std::max(V, 1)), order(std::max(V, 1)), off(r.count() + 1);
  std::vector<int64_t> start(std::max(V, 1));
  bx_placement out{dev.data(), start.data(), order.data(), off.data(), {0, 0, 0}, 0, {0}};
  if (bx_place(&f.g, &job, &out) != BX_OK) rethrow(out.status, bx_last_message());  // full text
  Placement p;
  p.algorithm = name;
  p.device_of.assign(dev.begin(), dev.begin() + V);
  p.start_us.assign(start.begin(), start.begin() + V);
  p.exec_order.assign(r.count(), {});
  for (int d = 0; d < r.count(); ++d) p.exec_order[d].assign(order.begin() + off[d], order.begin() + off[d + 1]);
  if (stats) *stats = PlacerStats{out.stats[0], out.stats[1], out.stats[2]};
  return p;
}
}  // namespace

Placement place_metf(const GroupedGraph& gg, const DeviceRoster& r, const CommModel& cm, PlacerStats* s) {
  return run(gg, r, cm, BX_ALGO_METF, nullptr, s, "m-etf");
}
Placement place_msct(const GroupedGraph& gg, const DeviceRoster& r, const CommModel& cm, const FavoriteMap& fav,
                     PlacerStats* s) {
  return run(gg, r, cm, BX_ALGO_MSCT, &fav, s, "m-sct");
}
Placement place_mtopo(const GroupedGraph& gg, const DeviceRoster& r, const CommModel& cm) {
  return run(gg, r, cm, BX_ALGO_MTOPO, nullptr, nullptr, "m-topo");
}
}  // namespace dagsched

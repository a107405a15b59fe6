// TEST INFRASTRUCTURE ONLY: drives the reference-side shim
// (integration/placers_b200.cpp, the INTEGRATION.md binding) with the
// reference's own types, next to the UNMODIFIED reference placer compiled
// from /root/reference with its place_* renamed ref_place_* (oracle/Makefile,
// target `shim`). Inputs: generate_graph (proj/src/generator.cpp:173) over
// the three families, singleton_groups / apply_colocation, uniform rosters
// at several capacity factors (including infeasible ones), both comm modes,
// m-TOPO / m-ETF / m-SCT (first-unclaimed-child favourites). Every case must
// give the same Placement + PlacerStats, or the same exception kind and
// what() text. Prints one JSON summary line; exit code 0 iff no mismatch.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "dagsched/cost_model.hpp"
#include "dagsched/errors.hpp"
#include "dagsched/generator.hpp"
#include "dagsched/graph.hpp"
#include "dagsched/lp.hpp"
#include "dagsched/placers.hpp"
#include "dagsched/transforms.hpp"

namespace dagsched {  // the reference placer, renamed at compile time
Placement ref_place_mtopo(const GroupedGraph& gg, const DeviceRoster& roster, const CommModel& cm);
Placement ref_place_metf(const GroupedGraph& gg, const DeviceRoster& roster, const CommModel& cm,
                         PlacerStats* stats);
Placement ref_place_msct(const GroupedGraph& gg, const DeviceRoster& roster, const CommModel& cm,
                         const FavoriteMap& fav, PlacerStats* stats);
}  // namespace dagsched

using namespace dagsched;

namespace {
struct Outcome {
  bool ok = false;
  int kind = -1;
  std::string what;
  Placement p;
  PlacerStats st;
};

Outcome call(const std::function<Placement(PlacerStats*)>& f) {
  Outcome o;
  try {
    o.p = f(&o.st);
    o.ok = true;
  } catch (const Error& e) {
    o.kind = static_cast<int>(e.kind());
    o.what = e.what();
  } catch (const std::exception& e) {
    o.kind = 99;
    o.what = e.what();
  }
  return o;
}

bool same(const Outcome& a, const Outcome& b, bool stats) {
  if (a.ok != b.ok) return false;
  if (!a.ok) return a.kind == b.kind && a.what == b.what;
  if (a.p.device_of != b.p.device_of || a.p.start_us != b.p.start_us || a.p.exec_order != b.p.exec_order)
    return false;
  return !stats || (a.st.discarded_pairs == b.st.discarded_pairs && a.st.excluded_devices == b.st.excluded_devices &&
                    a.st.awake_reservations == b.st.awake_reservations);
}

FavoriteMap first_unclaimed(const GroupedGraph& gg) {
  FavoriteMap f = FavoriteMap::none(gg.node_count());
  for (const MetaEdge& e : gg.edges)
    if (f.fav_child[e.src] < 0 && f.fav_parent[e.dst] < 0) {
      f.fav_child[e.src] = e.dst;
      f.fav_parent[e.dst] = e.src;
    }
  return f;
}
}  // namespace

int main() {
  int cases = 0, mismatches = 0, errors = 0;
  std::string first;
  const GraphFamily fams[3] = {GraphFamily::Branchy, GraphFamily::LayeredChain, GraphFamily::RandomDag};
  for (GraphFamily fam : fams) {
    for (int size : {40, 300, 1500}) {
      if (fam == GraphFamily::RandomDag && size > 300) continue;  // the generator is O(V^2)
      for (uint64_t seed : {1ull, 2ull}) {
        GenSpec spec;
        spec.family = fam;
        spec.node_count = size;
        spec.seed = seed;
        auto base = std::make_shared<const ProfiledGraph>(generate_graph(spec));
        GroupedGraph gg = seed == 1 ? singleton_groups(base) : apply_colocation(base);
        bytes_t total = 0, largest = 0;
        for (const MetaNode& m : gg.nodes) {
          const bytes_t r = m.perm_mem_bytes + m.out_mem_bytes + m.temp_mem_bytes;
          total += r;
          largest = std::max(largest, r);
        }
        const FavoriteMap fav = first_unclaimed(gg);
        for (int n : {1, 3, 8}) {
          for (double factor : {0.4, 1.05, 1.5}) {
            const bytes_t cap = static_cast<bytes_t>(std::ceil((double(total) / n + double(largest)) * factor));
            const DeviceRoster r = DeviceRoster::uniform(n, cap);
            for (CommMode mode : {CommMode::Parallel, CommMode::Sequential}) {
              const CommModel cm{12.5, 0.002, mode};
              for (int algo = 0; algo < 3; ++algo) {
                Outcome a, b;
                if (algo == 0) {
                  a = call([&](PlacerStats*) { return place_mtopo(gg, r, cm); });
                  b = call([&](PlacerStats*) { return ref_place_mtopo(gg, r, cm); });
                } else if (algo == 1) {
                  a = call([&](PlacerStats* s) { return place_metf(gg, r, cm, s); });
                  b = call([&](PlacerStats* s) { return ref_place_metf(gg, r, cm, s); });
                } else {
                  a = call([&](PlacerStats* s) { return place_msct(gg, r, cm, fav, s); });
                  b = call([&](PlacerStats* s) { return ref_place_msct(gg, r, cm, fav, s); });
                }
                ++cases;
                errors += !b.ok;
                if (!same(a, b, algo != 0)) {
                  if (!mismatches) {
                    char buf[512];
                    std::snprintf(buf, sizeof buf, "family %d size %d seed %d n %d factor %.2f mode %d algo %d: %s | %s",
                                  static_cast<int>(fam), size, static_cast<int>(seed), n, factor,
                                  static_cast<int>(mode), algo, a.ok ? "placed" : a.what.c_str(),
                                  b.ok ? "placed" : b.what.c_str());
                    first = buf;
                  }
                  ++mismatches;
                }
              }
            }
          }
        }
      }
    }
  }
  std::string esc;
  for (char ch : first) esc += (ch == '"' || ch == '\\') ? std::string("\\") + ch : std::string(1, ch);
  std::printf("{\"cases\": %d, \"reference_errors\": %d, \"mismatches\": %d, \"first_mismatch\": \"%s\"}\n", cases,
              errors, mismatches, esc.c_str());
  return mismatches ? 1 : 0;
}

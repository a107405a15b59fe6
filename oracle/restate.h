/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference hot path.
 *
 * This is the parity oracle: tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline leg may load it, the product never does. Each function cites
 * the reference lines it restates. It is pinned against the reference's own
 * known-answer tests (tests/test_oracle_kats.py) and against the compiled
 * reference itself (oracle/_ref, tests/test_oracle_vs_ref.py).
 *
 * Meta graph input: V nodes, E edges sorted by (src, dst) — the GroupedGraph
 * invariant of proj/include/dagsched/transforms.hpp:56 — with per-node
 * aggregates (compute, temp, perm, out). `first_id` (nullable) gives the base
 * id of each meta node's smallest member, used only in error messages.
 *
 * Return codes: 0 ok, 2 validation, 3 infeasible (ErrorKind, errors.hpp:12).
 */
#ifndef BAECHI_ORACLE_RESTATE_H
#define BAECHI_ORACLE_RESTATE_H
#include <stdint.h>

typedef struct {
  int32_t V, E;
  const int64_t *k, *temp, *perm, *out;
  const int32_t *esrc, *edst;
  const int64_t *ebytes;
  const int64_t *first_id; /* nullable */
} rs_graph;

int64_t rs_comm_time(double intercept, double per_byte, int64_t bytes, int *err);

/* algo: 0 m-topo, 1 m-etf, 2 m-sct (fav_child NULL = empty map). */
int rs_place(const rs_graph *g, int32_t algo, int32_t n, const int64_t *caps,
             double intercept, double per_byte, int32_t mode,
             const int32_t *fav_child, int32_t *device_of, int64_t *start,
             int32_t *exec_order, int32_t *exec_off, int64_t *stats3,
             char *msg, int msglen);

int rs_simulate(const rs_graph *g, int32_t n, const int64_t *caps,
                double intercept, double per_byte, int32_t mode,
                int32_t mem_mode, const int32_t *device_of,
                const int32_t *exec_order, const int32_t *exec_off,
                int64_t *makespan, int64_t *start, int64_t *dev3n,
                int64_t *xfer4, char *msg, int msglen);

int rs_round_extract(int32_t V, int32_t E, const int32_t *esrc,
                     const int32_t *edst, const double *x, double threshold,
                     int32_t *fav_child, int32_t *fav_parent, int32_t *stats2,
                     char *msg, int msglen);

int rs_topo_order(const rs_graph *g, int32_t *order, char *msg, int msglen);

#endif

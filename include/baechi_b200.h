/* baechi_b200.h — the drop-in C ABI of the B200 placement engine.
 *
 * Plain C, plain pointers and sizes; no CUDA or torch types cross this line.
 * Every entry point replaces one function of the reference C++ placer API
 * (namespace dagsched, /root/reference/proj/include/dagsched/<name>.hpp); the
 * citation sits above each declaration. INTEGRATION.md shows the bindings
 * (C++ shim, ctypes) a maintainer of the reference would add.
 *
 * Conventions:
 *  - status codes mirror dagsched::ErrorKind -> CLI exit code
 *    (errors.hpp:12-51, tools/dagsched.cpp:350-368): 0 ok, 2 validation,
 *    3 infeasible, 4 solver; 5 = CUDA/runtime failure (no reference analogue).
 *    Nothing throws across the ABI; `msg` receives the reference's message.
 *  - graphs are META graphs (GroupedGraph, transforms.hpp:34-53): V meta
 *    nodes numbered as the transforms number them, E meta edges sorted by
 *    (src, dst) and unique, plus the adjacency GroupedGraph carries
 *    (in_edges / out_edges as CSR of edge ids, ascending).
 *  - all costs are int64 microseconds / bytes; placements are bit-exact with
 *    the reference (device_of, exec_order, start_us, PlacerStats).
 *  - inputs are caller-owned and read-only; outputs are caller-allocated.
 *  - there is no CPU fallback: without a CUDA device every compute entry
 *    point returns 5 with a message saying so.
 */
#ifndef BAECHI_B200_H
#define BAECHI_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define BX_OK 0
#define BX_VALIDATION 2
#define BX_INFEASIBLE 3
#define BX_SOLVER 4
#define BX_RUNTIME 5

#define BX_ALGO_MTOPO 0
#define BX_ALGO_METF 1
#define BX_ALGO_MSCT 2

#define BX_COMM_SEQUENTIAL 0 /* CommMode::Sequential (cost_model.hpp:11) */
#define BX_COMM_PARALLEL 1   /* CommMode::Parallel */

#define BX_MEM_GRAPH_STATIC 0        /* MemoryMode::GraphStatic (cost_model.hpp:13) */
#define BX_MEM_TRAINING_PERSISTENT 1 /* MemoryMode::TrainingPersistent */

/* GroupedGraph (transforms.hpp:34-53) flattened. in_edge lists, per meta
 * node, the ids of its incoming meta edges in ascending order
 * (GroupedGraph::in_edges); out-edges are contiguous because edges are
 * sorted by src, so out_off alone describes GroupedGraph::out_edges.
 * first_id (nullable) is the external id of each meta node's smallest
 * member, used only in error messages (simulator.cpp:54-56). */
typedef struct {
  int32_t V, E;
  const int64_t *compute_us, *temp_bytes, *perm_bytes, *out_bytes; /* [V] */
  const int32_t *esrc, *edst;                                      /* [E] */
  const int64_t *tensor_bytes;                                     /* [E] */
  const int32_t *in_off, *in_edge;                                 /* [V+1], [E] */
  const int32_t *out_off;                                          /* [V+1] */
  const int64_t *first_id;                                         /* [V] or NULL */
} bx_graph;

/* CommModel (cost_model.hpp:19-24). */
typedef struct {
  double intercept_us, us_per_byte;
  int32_t mode; /* BX_COMM_* */
} bx_comm;

/* One placement problem: place_mtopo / place_metf / place_msct
 * (placers.hpp:73-89) of `graph` on a roster of n devices. */
typedef struct {
  int32_t graph;               /* index into the plan's graph array */
  int32_t algo;                /* BX_ALGO_* */
  int32_t n;                   /* DeviceRoster::count() */
  const int64_t *capacity;     /* [n] DeviceRoster capacities (bytes) */
  bx_comm cm;
  const int32_t *fav_child;    /* m-sct FavoriteMap::fav_child [V]; NULL = empty map */
  int32_t fav_len;             /* length of fav_child as given (0 or V), for the size check */
} bx_job;

/* Placement (placers.hpp:25-32) + PlacerStats (:34-38), caller-allocated. */
typedef struct {
  int32_t *device_of;   /* [V] */
  int64_t *start_us;    /* [V] */
  int32_t *exec_order;  /* [V]  concatenated per-device lists */
  int32_t *exec_off;    /* [n+1] */
  int64_t stats[3];     /* discarded_pairs, excluded_devices, awake_reservations */
  int32_t status;       /* BX_* of this job */
  char msg[256];        /* reference error text when status != 0 */
} bx_placement;

/* SimReport (simulator.hpp:25-34), caller-allocated. */
typedef struct {
  int64_t makespan_us;
  int64_t *start_us;        /* [V] */
  int64_t *peak_bytes;      /* [n] DeviceReport::peak_bytes */
  int64_t *busy_us;         /* [n] */
  int64_t *idle_us;         /* [n] */
  int64_t transfer_count, transfer_bytes, duplicate_transfers, cache_hits;
  int32_t status;
  char msg[256];
} bx_sim_report;

/* ---- library ---------------------------------------------------------- */
const char *bx_version(void);
/* Text of the last CUDA launch failure seen by this thread ("" if none). */
const char *bx_last_error(void);
/* Full reference error text of this thread's last bx_place call (msg[256]
 * holds a prefix; a CycleError lists every residue group id). */
const char *bx_last_message(void);
/* Number of CUDA devices visible (0 on a CPU-only host). */
int bx_device_count(void);

/* comm_time (cost_model.cpp:30-36): round_half_up(intercept + per_byte*bytes)
 * with separately rounded multiply and add (no FMA). Host-side scalar
 * helper used by the C++ shim; the kernels compute the same thing on device. */
int bx_comm_time(const bx_comm *cm, int64_t bytes, int64_t *out_us);

/* Builds GroupedGraph adjacency for a meta edge list already sorted by
 * (src, dst): in_off/in_edge and out_off (transforms.cpp:169-223 fills the
 * same lists). Host-side ingest helper, O(V+E). */
int bx_build_adjacency(int32_t V, int32_t E, const int32_t *esrc,
                       const int32_t *edst, int32_t *in_off, int32_t *in_edge,
                       int32_t *out_off, char *msg, int msglen);

/* ---- ingest: base graph -> GroupedGraph (host C++) ----------------------
 * A ProfiledGraph (graph.hpp:10-40) as arrays. Colocation groups are given
 * as integer labels (equal label = same colocation_group string; -1 none);
 * coplace_pair as has_pair + peer id. Node/edge order is free. */
typedef struct {
  int32_t nodes;
  const int64_t *id, *compute_us, *temp_bytes, *perm_bytes, *out_bytes; /* [nodes] */
  const int32_t *coloc_label;   /* [nodes] or NULL */
  const uint8_t *has_pair;      /* [nodes] or NULL */
  const int64_t *coplace_peer;  /* [nodes] or NULL */
  int32_t edges;
  const int64_t *src, *dst, *tensor_bytes; /* [edges], node ids */
} bx_base_graph;

/* Base-node view of a grouping (GroupedGraph::group_of / MetaNode::members,
 * MetaEdge::base_count). */
typedef struct {
  int32_t base_nodes;
  const int64_t *base_ids;        /* [base_nodes] ascending (make_graph order) */
  const int32_t *group_of;        /* [base_nodes] base index -> meta index */
  const int32_t *members;         /* concatenated base indices per meta node */
  const int32_t *member_off;      /* [V+1] */
  const int32_t *edge_base_count; /* [E] */
} bx_grouping;

#define BX_PIPE_SINGLETON (-1)    /* singleton_groups only */
#define BX_PIPE_COLOCATION 0      /* apply_colocation */
#define BX_PIPE_COPLACEMENT 2     /* + apply_coplacement */
#define BX_PIPE_FUSION 4          /* + fuse_operators */

typedef struct bx_grouped bx_grouped;

/* make_graph (graph.cpp:99-194) then build_grouped (bench.cpp:43-49):
 * singleton groups, colocation (transforms.cpp:329-351), optional
 * co-placement (:353-388) and fusion (:390-444). Validation / CycleError
 * texts are the reference's; status BX_VALIDATION on failure. */
int bx_grouped_create(const bx_base_graph *base, int32_t pipeline, bx_grouped **out, char *msg, int msglen);
/* Views into the grouped graph (valid until destroy): the meta graph ready
 * for bx_plan_create / bx_place, and the base-node grouping. */
int bx_grouped_view(const bx_grouped *grouped, bx_graph *meta, bx_grouping *grouping);
void bx_grouped_destroy(bx_grouped *grouped);

/* ---- plans: device-resident batches of placement problems --------------
 * A plan owns device copies of `ngraphs` graphs and `njobs` jobs plus the
 * scheduling workspace. It remembers the caller's host pointers, so
 * bx_plan_upload / bx_plan_download re-copy inputs and outputs (the
 * end-to-end path) while bx_plan_place runs on device-resident data only.
 * `device` selects the CUDA device the plan lives on. */
typedef struct bx_plan bx_plan;

int bx_plan_create(int32_t ngraphs, const bx_graph *graphs, int32_t njobs,
                   const bx_job *jobs, int32_t device, bx_plan **out,
                   char *msg, int msglen);

/* Kernel-dispatch options of a plan (bx_plan_create uses the defaults).
 * Results never depend on them — every kernel is bit-exact — only speed
 * does; tests use them to drive each kernel over the same cases. Zero-
 * initialise and set what you need; 0 / -1 mean "default". */
typedef struct {
  int32_t no_small_frontier; /* 1: never try the small-frontier kernel (K2s) */
  int32_t wide_min_vn;       /* >= 0: V*n from which list jobs take the CTA-wide kernels; -1 default */
  int32_t wide_max_jobs;     /* > 0: at most this many CTA-wide jobs (default 120) */
  int32_t list_len;          /* 4/8/16/32: round-kernel column list length; 0 default */
  int32_t profile;           /* 1: clock64-instrumented placer (bx_plan_profile) */
  int32_t sim_heap_cap;      /* >= 0: shared-memory event heap slice of K4; -1 default */
  int32_t sim_trace;         /* 1: simulations record SimOptions::record_trace events (bx_plan_sim_trace) */
} bx_plan_options;

int bx_plan_create_ex(int32_t ngraphs, const bx_graph *graphs, int32_t njobs,
                      const bx_job *jobs, int32_t device,
                      const bx_plan_options *options, bx_plan **out,
                      char *msg, int msglen);
void bx_plan_destroy(bx_plan *plan);

/* Host -> device copy of every graph/job input, enqueued on `stream`
 * (a cudaStream_t passed as void*; NULL = legacy default stream). */
int bx_plan_upload(bx_plan *plan, void *stream);

/* Ingest (K1) + placement (K2) of every job, device-resident, on `stream`.
 * Runs the reference's validation order per job: fav size (place_msct,
 * placers.cpp:304-310), roster (:19-29), m-topo cap (:327-335), acyclicity
 * (meta_topo_order, transforms.cpp:446-479), then the placer. Asynchronous;
 * per-job status lands on the device and is read by bx_plan_download. */
int bx_plan_place(bx_plan *plan, void *stream);

/* Device -> host copy of every job's placement into `out[njobs]`
 * (caller-allocated arrays sized by each job's V and n). Synchronises
 * `stream`. Returns BX_OK if the copy worked; per-job status is in out[i]. */
int bx_plan_download(bx_plan *plan, void *stream, bx_placement *out);
/* The same device->host copy of the output region into the plan's pinned
 * mirror, enqueued on `stream` only (no wait, no decode): for pipelined
 * callers that keep two plans in flight. */
int bx_plan_download_async(bx_plan *plan, void *stream);

/* The outputs of every job live in one device region that bx_plan_download
 * copies (one cudaMemcpyAsync) into a pinned host mirror owned by the plan;
 * `out` may be NULL to skip the per-job copies into caller buffers. This
 * returns a zero-copy view of job `job` inside that mirror (valid until the
 * next download or destroy). */
int bx_plan_result_view(bx_plan *plan, int32_t job, bx_placement *view);
/* Full error text of a job after bx_plan_download (msg[256] holds a prefix):
 * copies up to buflen-1 bytes + NUL, returns the full length (-1: no result). */
int64_t bx_plan_message(const bx_plan *plan, int32_t job, char *buf, int64_t buflen);

/* Number of kernel launches the last bx_plan_place issued. */
int bx_plan_launch_count(const bx_plan *plan);

/* Which kernel placed job `job` in the last bx_plan_place (waits for it). */
#define BX_KERNEL_NONE (-1)          /* host validation failed: never launched */
#define BX_KERNEL_MTOPO 0            /* k_place_topo */
#define BX_KERNEL_WARP 1             /* k_place_list<1>: one warp per problem */
#define BX_KERNEL_ROUNDS 2           /* k_place_rounds: CTA per problem, parallel comm */
#define BX_KERNEL_CTA_SEQ 3          /* k_place_list<8>: CTA per problem, sequential comm */
#define BX_KERNEL_SMALL_FRONTIER 4   /* k_place_small: one warp, shared-memory state (smallsched.cu) */
#define BX_KERNEL_SEQ_SMALL 5        /* k_place_seq_small: one warp, sequential comm, small frontier (seqsmall.cu) */
int bx_plan_job_kernel(bx_plan *plan, int32_t job);

/* Device time (ms) of the placer kernel(s) of the last bx_plan_place,
 * measured with CUDA events on the plan's stream; waits for it. */
float bx_plan_kernel_ms(bx_plan *plan);
/* The same for each of the last `count` bx_plan_place calls (at most 64 are
 * kept), oldest first, without synchronising between them: a timed loop of
 * places reads its per-step kernel times afterwards. Returns how many. */
int bx_plan_kernel_times(bx_plan *plan, int32_t count, float *ms);

/* The device-resident output region of the plan (every job's placement and
 * status, the bytes bx_plan_download copies) and, per job, the byte offsets
 * inside it of device_of, start_us, exec_order, exec_off, stats[3] and the
 * status record (int32 status, int32 code, 4 x int64 detail). A sweep
 * gathers these regions from every rank over NCCL. */
int bx_plan_output_region(const bx_plan *plan, void **dev, int64_t *bytes);
int bx_plan_job_outputs(const bx_plan *plan, int32_t job, int64_t *offs6);

/* Per-step latency breakdown of job `job` (plans created with
 * bx_plan_options.profile = 1 run a clock64-instrumented placer):
 * 16 int64 = SM cycles in rescan, argmin, rekey, discard, commit, remove,
 * ready, rows, cache, insert, emit, then counts steps, commits, rescans,
 * and the total cycles of the job. */
int bx_plan_profile(bx_plan *plan, int32_t job, int64_t *out16);

/* simulate (simulator.cpp:273-278) of every job's current device-resident
 * placement, in `mem_mode`: K4f (FIFO walkers + max-plus scans) for parallel
 * comm without zero-duration nodes, K4 (the reference's event heap order)
 * otherwise. Device-resident; use bx_plan_sim_download for the reports. */
int bx_plan_simulate(bx_plan *plan, int32_t mem_mode, void *stream);
int bx_plan_sim_download(bx_plan *plan, void *stream, bx_sim_report *out);

/* ---- one-shot entry points (host buffers in, host buffers out) ---------
 * bx_place == place_mtopo / place_metf / place_msct (placers.hpp:73-89). */
int bx_place(const bx_graph *graph, const bx_job *job, bx_placement *out);

/* bx_simulate == simulate (simulator.hpp:53-55) of an externally given
 * placement (device_of [V], exec_order/exec_off per device). */
int bx_simulate(const bx_graph *graph, int32_t n, const int64_t *capacity,
                const bx_comm *cm, int32_t mem_mode, const int32_t *device_of,
                const int32_t *exec_order, const int32_t *exec_off,
                bx_sim_report *out);
/* bx_simulate with plan options (tests: sim_heap_cap). */
int bx_simulate_ex(const bx_graph *graph, int32_t n, const int64_t *capacity,
                   const bx_comm *cm, int32_t mem_mode, const int32_t *device_of,
                   const int32_t *exec_order, const int32_t *exec_off,
                   const bx_plan_options *options, bx_sim_report *out);

/* LpSolution (lp.hpp:47-53) bookkeeping + SctLp row-class counts (:33-38). */
typedef struct {
  int32_t iterations;
  double rel_gap;
  double w;            /* unscaled objective after re-tightening the starts */
  int32_t num_rows, completion_rows, precedence_rows, child_rows, parent_rows, bound_rows;
  /* K5 solver diagnostics: host build (rows, ordering, symbolic factor) and
   * device IPM time, factor nonzeros, right-looking update pairs (0 = the
   * factorization walks target columns instead of a precomputed map) */
  double host_ms, device_ms;
  int64_t factor_nnz, update_pairs;
} bx_lp_info;

/* bx_lp_solve == build_lp + solve_relaxed (lp.hpp:45-59, lp.cpp:14-278) on a
 * meta graph: the same Mehrotra IPM (scaling, start point, eta, stopping
 * rule, 200-iteration cap), the whole IPM loop on the GPU in one CTA with a
 * hand-written sparse Cholesky of the normal equations (minimum-degree
 * ordering, K5). x [E] (clipped to [0,1]) and s [V] (nullable) are the
 * unscaled solution. BX_SOLVER with the reference's text on failure. */
int bx_lp_solve(const bx_graph *graph, const bx_comm *cm, double tolerance, double *x, double *s,
                bx_lp_info *info, char *msg, int msglen);

/* oracle_makespan (oracle.hpp:29-34, oracle.cpp:17-212): the exact minimum
 * makespan over every canonical device assignment and every DAG-consistent
 * per-device execution order, each scored by the GPU simulator in batches.
 * capacity < 0: none (OracleLimits / prepare() limits and error texts;
 * BX_INFEASIBLE when nothing fits or the instance is too large). */
int bx_oracle_makespan(const bx_graph *graph, int32_t n, const bx_comm *cm, int64_t capacity, int32_t mem_mode,
                       int32_t max_nodes, int32_t max_devices, int64_t max_extensions, int64_t *out_us,
                       char *msg, int msglen);

/* bx_round_extract == round_and_extract (lp.hpp:88-90, lp.cpp:280-326) on
 * the device (K3): x[E] per meta edge, threshold in (0, 0.5).
 * stats2 = {favorite_edges, repaired_nodes}. */
int bx_round_extract(int32_t V, int32_t E, const int32_t *esrc,
                     const int32_t *edst, const double *x, double threshold,
                     int32_t *fav_child, int32_t *fav_parent, int32_t *stats2,
                     char *msg, int msglen);

/* ---- partial-schedule queries ---------------------------------------------
 * PlacerState (placers.hpp:49-60) flattened: mode is PlacerState::mode (the
 * queue discipline of the estimate), cache_arrival is [V*n] row-major by
 * meta node, -1 = absent. */
typedef struct {
  int32_t V, n, mode;             /* mode: BX_COMM_* */
  const int64_t *dev_free;        /* [n] */
  const int64_t *xfer_tail;       /* [n] */
  const int32_t *device_of;       /* [V] -1 = unplaced */
  const int64_t *finish_us;       /* [V] */
  const int64_t *cache_arrival;   /* [V*n] */
} bx_placer_state;

/* schedulable_time (placers.hpp:66-67, placers.cpp:43-91) of `count` (node,
 * device) queries against one partial schedule, evaluated on the GPU (one
 * thread per query): out[i] = earliest start of node[i] on device[i]. The
 * state is not modified (the sequential-mode queue tails are folded on a
 * private copy, as the reference's estimate does). In sequential mode an
 * uncached remote parent must be placed (the reference indexes its queue). */
int bx_schedulable_time(const bx_graph *graph, const bx_comm *cm, const bx_placer_state *state, int32_t count,
                        const int32_t *node, const int32_t *device, int64_t *out, char *msg, int msglen);

/* critical_path_us (simulator.cpp:296-309): the compute-weighted longest
 * path of the meta graph (a level-synchronous peel on the GPU). Cyclic
 * graphs fail with meta_topo_order's CycleError text (BX_VALIDATION). */
int bx_critical_path_us(const bx_graph *graph, int64_t *out_us, char *msg, int msglen);

/* ---- simulator trace (SimOptions::record_trace, simulator.hpp:19-37) ------ */
#define BX_TRACE_START 0
#define BX_TRACE_FINISH 1
#define BX_TRACE_XFER_BEGIN 2
#define BX_TRACE_XFER_END 3
typedef struct {
  int64_t time_us;
  int32_t device;
  int32_t event;   /* BX_TRACE_* ("start" | "finish" | "xfer_begin" | "xfer_end") */
  int64_t node;    /* base node id of the meta node's first member */
} bx_trace_event;

/* bx_simulate with record_trace: `trace` receives SimReport::trace in the
 * reference's processing order (at most trace_cap events; *trace_len = the
 * number recorded, 2V + 2E bounds it). */
int bx_simulate_trace(const bx_graph *graph, int32_t n, const int64_t *capacity, const bx_comm *cm,
                      int32_t mem_mode, const int32_t *device_of, const int32_t *exec_order,
                      const int32_t *exec_off, bx_sim_report *out, bx_trace_event *trace, int64_t trace_cap,
                      int64_t *trace_len);
/* The trace of job `job` of a plan created with bx_plan_options.sim_trace. */
int bx_plan_sim_trace(bx_plan *plan, int32_t job, bx_trace_event *out, int64_t cap, int64_t *len);
/* trace_to_csv (simulator.cpp:311-324): header "time_us,device,event,node",
 * rows stable-sorted by time. Writes a NUL-terminated string into buf when
 * buflen >= *needed (else BX_VALIDATION and only *needed is set). */
int bx_trace_to_csv(const bx_trace_event *trace, int64_t count, char *buf, int64_t buflen, int64_t *needed);

/* ---- interchange IO (host C++, csrc/jsonio.cpp) ----------------------------
 * JSON texts are read in one schema-directed pass (no DOM) with the
 * reference's validation order and messages; emitted texts are
 * byte-identical to nlohmann's dump(2) + "\n" as the reference writes them.
 * Emitters write a NUL-terminated string into buf when buflen >= *needed,
 * else return BX_VALIDATION with only *needed set. */

/* parse_comm_model / load_comm_model / save_comm_model (cost_model.cpp:71-134). */
int bx_comm_model_parse(const char *text, int64_t len, bx_comm *out, char *msg, int msglen);
int bx_comm_model_load(const char *path, bx_comm *out, char *msg, int msglen);
int bx_comm_model_to_json(const bx_comm *cm, char *buf, int64_t buflen, int64_t *needed);

/* parse_graph / load_graph (graph.cpp:196-281) up to, not including,
 * make_graph: the parsed base graph (file order) with its node names and
 * colocation groups as labels (labels index the sorted distinct group
 * strings). bx_grouped_create runs make_graph + the transforms on the view. */
typedef struct bx_json_graph bx_json_graph;
int bx_graph_parse(const char *text, int64_t len, bx_json_graph **out, char *msg, int msglen);
int bx_graph_load(const char *path, bx_json_graph **out, char *msg, int msglen);
int bx_json_graph_view(const bx_json_graph *g, bx_base_graph *base, const char *const **names,
                       const char *const **groups, int32_t *ngroups);
void bx_json_graph_destroy(bx_json_graph *g);
/* graph_to_json (graph.cpp:283-309) of a ProfiledGraph: nodes by ascending
 * id, edges by (src, dst). names [nodes] / groups [labels] may be NULL. */
int bx_graph_to_json(const bx_base_graph *g, const char *const *names, const char *const *groups, char *buf,
                     int64_t buflen, int64_t *needed);

/* placement_to_json / placement_from_json (placers.cpp:367-432). The
 * grouping is the GroupedGraph's (bx_grouped_view). to_json writes one row
 * per base member of every meta node in exec order with its simulated
 * start; from_json fills device_of/start_us [V] and exec lists (file order). */
int bx_placement_to_json(const bx_grouping *grouping, const char *algorithm, int32_t n, const int32_t *exec_order,
                         const int32_t *exec_off, const int64_t *sim_start_us, int64_t makespan_us,
                         const int64_t *peak_bytes, char *buf, int64_t buflen, int64_t *needed);
int bx_placement_from_json(const bx_grouping *grouping, int32_t V, const char *text, int64_t len, int32_t n,
                           char *algorithm, int algolen, int32_t *device_of, int64_t *start_us,
                           int32_t *exec_order, int32_t *exec_off, char *msg, int msglen);

/* Binary CSR sidecar of a meta graph: save, and load into an owned copy
 * whose bx_graph view feeds bx_plan_create directly (adjacency checked). */
typedef struct bx_bin_graph bx_bin_graph;
int bx_graph_save_bin(const bx_graph *graph, const char *path, char *msg, int msglen);
int bx_graph_load_bin(const char *path, bx_bin_graph **out, bx_graph *view, char *msg, int msglen);
void bx_bin_graph_destroy(bx_bin_graph *g);

#ifdef __cplusplus
}
#endif
#endif /* BAECHI_B200_H */

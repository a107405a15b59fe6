// Device-side data layout shared by the ingest (K1), placer (K2), extract
// (K3) and simulator (K4) kernels. Everything is int64 microseconds / bytes,
// so every kernel result is bit-exact with the reference.
//
// HBM layout per plan (one cudaMalloc pool, 256-byte aligned sub-arrays):
//   graph arrays  (read-only, shared by every job on that graph)
//     k, temp, perm, out, need        int64 [V]
//     esrc, edst(=out-CSR dst list)   int32 [E]   ascending (src, dst)
//     ebytes                          int64 [E]
//     in_off / out_off                int32 [V+1]
//     in_edge, in_src                 int32 [E]   in-CSR, ascending src
//     need_order                      int32 [V]   ascending need (min remaining)
//   prep arrays (per distinct (graph, comm model))
//     in_c                            int64 [E]   comm_time per in-CSR slot
//   job workspace (per job)
//     K, cache                        int64 [V*n] key lower bound / arrival
//     dead                            uint8 [V*n]
//     pending, alive, ready, rpos,
//     cseq, nc                        int32 [V]
//     finish, urgent                  int64 [V]
//     scratch tails                   int64/int32 [32*n] per warp lane
//   job outputs
//     device_of int32 [V], start int64 [V], exec_order int32 [V],
//     exec_off int32 [n+1], stats int64 [3], err (status, code, a, b)
#pragma once
#include <cstdint>

namespace bx {

constexpr int kOk = 0;
constexpr int kValidation = 2;
constexpr int kInfeasible = 3;
constexpr int kRuntime = 5;

// Device-side error codes; the host formats the reference's message text.
enum ErrCode : int32_t {
  E_NONE = 0,
  E_FITS_NONE = 1,   // "node j fits on no device"              placers.cpp:173-179
  E_NO_PAIR = 2,     // "no schedulable (node, device) pair..."  placers.cpp:190-192
  E_CYCLE = 3,       // CycleError from meta_topo_order          transforms.cpp:446-479
  E_NEG_BYTES = 4,   // "comm_time: negative byte count"         cost_model.cpp:31-33
  E_TOPO_CAP = 5,    // m-topo cap > smallest capacity           placers.cpp:327-335
  E_SIM_MEMORY = 6,  // simulator memory violation               simulator.cpp:66-76
  E_SIM_DEADLOCK = 7,// simulator deadlock                       simulator.cpp:234-246
  E_SIM_STALL = 8,   // "deadlock: simulation stalled"
  E_SIM_EXEC = 9,    // "exec_order disagrees with assignments"   simulator.cpp:87-89
  E_SIM_ONCE = 10,   // "placement must assign every node exactly once" :92-95
  E_HOST = 11,       // host-side validation failed (message kept by the plan)
};

struct DErr {
  int32_t status;
  int32_t code;
  int64_t a, b, c, d;
};

struct DGraph {
  int32_t V, E;
  const int64_t *k, *temp, *perm, *outb;
  const int32_t *esrc, *edst;
  const int64_t *ebytes;
  const int32_t *in_off, *in_edge, *out_off;
  // derived by K1 (graph level)
  int64_t *need;
  int32_t *need_order;  // node indices by ascending (need, index)
  int32_t *iota;        // sort scratch
  int64_t *need_keys;   // sort scratch
  int32_t *in_src;
  int32_t *inpos;       // [E] in-CSR slot of each edge (out-CSR order = edge order)
  int32_t *indeg_left;  // Kahn residue (cycle message)
  int32_t *flags;       // [0] peeled count, [1] negative-bytes flag, [2] negative compute time
  int64_t *ksum;        // sum of compute times (K2s int32 time bound)
};

struct DPrep {
  int32_t graph;
  int32_t first;  // 1: the first prep of its graph derives the graph-level arrays
  double ic, pb;
  int64_t *in_c;   // [E] comm_time of the in-CSR slot's edge
  int64_t *cmax;   // max_comm_time (cost_model.cpp:234-240)
  // K2s (small-frontier kernel) extras, filled by k_prep_small when a job needs them
  int32_t *in_c32;    // [E] in_c as int32 (valid when *cbad == 0)
  int32_t *nu;        // [V] index of a producer whose out-edges carry different comm times, else -1
  int32_t *nu_count;  // number of such producers
  int32_t *cbad;      // some comm time outside [0, 2^16 - 1)
  int4 *node_pack;    // [V] in_b, out_b, in_cnt | out_cnt << 16, k (int32) (needs from the graph's need[])
  uint2 *in_pack;     // [E] per in-CSR slot: parent, (nu(parent) + 1) << 16 | comm time
};

struct DJob {
  int32_t graph, prep, algo, n, mode, skip;
  const int64_t *cap;
  const int32_t *fav;
  // workspace
  int64_t *K, *cache;
  uint8_t *dead;
  int32_t *pending, *alive, *ready, *rpos, *cseq, *nc;
  int64_t *finish, *urgent;
  int64_t *sc_val;
  int32_t *sc_gen;
  int32_t *pdev;  // [E] per in-CSR slot: device of the (placed) parent
  // round kernel only (parallel comm mode, one CTA per problem): double
  // buffers for slot compaction and the per-round work lists
  int64_t *K2, *urgent2;
  int32_t *ready2, *alive2, *ncw, *newl;
  int64_t *pfin;  // [E] per in-CSR slot: finish time of the parent
  // outputs
  int32_t *device_of;
  int64_t *start;
  int32_t *exec_order, *exec_off;
  int64_t *stats;
  DErr *err;
  int64_t *prof;  // [kProfSlots] per-phase SM cycles when built with profiling, else null
  // K2s: set to 1 when the small-frontier kernel placed the job (or reported
  // its error); the general kernels then skip it. Null: not a K2s job.
  int32_t *sdone;
  int32_t nucap;  // K2s shared-memory slots reserved for non-uniform producers
  int32_t nocache;  // parallel comm, every producer uniform in bytes: no cache (Ctx::nocache)
  int32_t maxin;  // largest in-degree of the graph (K2s list sizing)
};

// One chunk of a per-step workspace fill (k_fill); at most kFillChunk bytes,
// 4-byte aligned; byte i = byte (i mod 4) of the little-endian `word`.
struct FillChunk {
  void *ptr;
  uint32_t bytes;
  uint32_t word;
};
constexpr size_t kFillChunk = 64 * 1024;

// Per-step latency breakdown slots (clock64 cycles summed over the run, lane 0).
enum ProfSlot : int {
  P_RESCAN = 0, P_ARGMIN, P_REKEY, P_DISCARD, P_COMMIT, P_REMOVE, P_READY, P_ROWS, P_CACHE, P_INSERT, P_EMIT,
  P_STEPS, P_COMMITS, P_RESCANS, P_TOTAL, kProfSlots = 16
};

// Simulator job (K4) — reads a placement (device_of / exec lists).
struct DSim {
  int32_t graph, n, mode, mem_mode;
  double ic, pb;
  const int64_t *cap;
  const int32_t *device_of, *exec_order, *exec_off;
  // workspace
  int64_t *mem, *peak, *xfree;      // [n]
  int32_t *qpos;                    // [n]
  uint8_t *busy;                    // [n]
  int32_t *consumers_left;          // [V]
  uint8_t *finished, *start_q;      // [V]
  uint8_t *resident, *sent;         // [V*n]
  int64_t *heap_t;                  // event heap: time
  int64_t *heap_k;                  // packed (kind, a, b)
  int64_t heap_cap;
  int32_t *seen;                    // [V] validation
  int64_t *dest_bytes;              // [n]
  int32_t *dest_cnt;                // [n]
  // dataflow (parallel comm mode) workspace, K4f
  int32_t *pos;                     // [V] position of a node in its device's exec_order
  int32_t *psrc;                    // [E] parent of each in-CSR slot
  int64_t *cx;                      // [E] arrival delay per in-CSR slot (-1 same device, -2 never)
  int64_t *fin;                     // [V] finish time, -1 until published
  int64_t *sx;                      // [V] start time per exec slot
  int64_t *bucket;                  // [V] output bytes freed before each exec slot's start
  int64_t *mb;                      // [V*n] max bytes per (producer, consumer device); sequencer:
                                    //     transfer time, then -2 - arrival once sent
  uint8_t *first;                   // [E] edge opens its (producer, device) transfer
  unsigned long long *flow8;        // [8] zero-k, bad exec, bad once, transfers, bytes, remote edges
  int32_t *rcnt;                    // [V] remote parents per node (bit 30: never ready)
  int32_t *rp_off;                  // [V+1] remote-parent lists by FIFO slot
  int32_t *rp_src;                  // [E] remote parent
  int64_t *rp_c;                    // [E] its arrival delay
  int64_t *kx;                      // [V] compute time by FIFO slot (-1: never ready)
  int64_t *dv;                      // [4n] per device: peak, violation t, node, memory
  int32_t *ninp;                    // [V] K4: inputs of a node not yet resident on its device
                                    //     sequencer: remote destination mask
  // SimOptions::record_trace (simulator.hpp:37): K4 appends (t, device,
  // event, meta) per event in processing order; null = no trace
  int64_t *trace;
  int64_t trace_cap;                // events the buffer holds
  unsigned long long *trace_n;      // events recorded
  // outputs
  int64_t *start;                   // [V]
  int64_t *dev3n;                   // [3n] peak, busy, idle
  int64_t *xfer4;                   // count, bytes, duplicates, cache hits
  int64_t *makespan;
  DErr *err;
};

// K3 arguments (round_and_extract).
struct XCtx {
  int V, E;
  const int32_t *esrc, *edst;
  const double *x;
  double thr;
  unsigned long long *src_min, *dst_min;  // [V] init ~0
  int32_t *src_peer, *dst_peer;           // [V] init INT_MAX
  int32_t *cnt_src, *cnt_dst;             // [V] init 0
  int32_t *best_edge;                     // [V] init -1
  int32_t *fav_child, *fav_parent;        // [V] init -1
  int32_t *stats2;                        // [2] init 0
};

// comm_time with the reference's exact double arithmetic: multiply, then
// add, each rounded once (no FMA contraction), then floor(v + 0.5).
__host__ __device__ inline int64_t comm_time_exact(double ic, double pb, int64_t bytes) {
#ifdef __CUDA_ARCH__
  double v = __dadd_rn(ic, __dmul_rn(pb, static_cast<double>(bytes)));
  return static_cast<int64_t>(floor(__dadd_rn(v, 0.5)));
#else
  volatile double prod = pb * static_cast<double>(bytes);
  volatile double sum = ic + prod;
  volatile double half = sum + 0.5;
  return static_cast<int64_t>(__builtin_floor(half));
#endif
}

}  // namespace bx

// The C ABI (include/baechi_b200.h): plans of device-resident placement
// problems, their uploads/downloads, kernel launches and the reference's
// error texts. Host-side C++; the compute is K1-K4 on the device.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <new>
#include <string>
#include <tuple>
#include <vector>

#include "../../include/baechi_b200.h"
#include "arena.hpp"
#include "bx_device.cuh"

namespace bx {
void launch_prep_all(const DGraph *graphs_dev, const DPrep *preps_dev, int nprep, int max_ev, cudaStream_t s);
void launch_fill(const FillChunk *table, int n, cudaStream_t s);
void launch_kahn(DGraph *graphs_dev, int32_t *const *queues_dev, int ngraphs, cudaStream_t s);
cudaError_t sort_needs_all(void *tmp, size_t &tmp_bytes, const int64_t *need, int64_t *keys_out, const int32_t *iota,
                           int32_t *order_out, int total, int nseg, const int32_t *seg_off, cudaStream_t s);
void launch_extract(const XCtx &c, cudaStream_t s);
void launch_placers(const DJob *jobs, const int32_t *order, int n_small, int n_etf, int n_bpar, int n_bseq,
                    int njobs, const DGraph *graphs, const DPrep *preps, int maxn, bool prof,
                    int list_len, cudaStream_t s_small, cudaStream_t s_big);
void launch_simulate(const DSim *sims, int nsims, const DGraph *graphs, int maxn, int force_cap, cudaStream_t s);
void launch_prep_small(const DGraph &g, const DPrep &pr, cudaStream_t s);
void launch_small_frontier(const DJob *jobs, const int32_t *order, const int *cnt, const DGraph *graphs,
                           const DPrep *preps, const size_t *smem, bool prof, cudaStream_t s);
size_t small_smem_bytes_host(int V, int n, int nucap, int nccap);
size_t small_pend_bytes_host(int V, int n, int nucap, int nccap, int maxin);
size_t seq_small_smem_bytes_host(int n, int V, int maxin);
void launch_seq_small(const DJob *jobs, const int32_t *order, int nj, const DGraph *graphs, const DPrep *preps,
                      size_t smem, bool prof, cudaStream_t s);
size_t topo_smem_bytes(int V, size_t limit);
void launch_topo(const DJob *jobs, int njobs, const DGraph *graphs, const DPrep *preps, size_t smem_bytes,
                 cudaStream_t s);
}  // namespace bx

using namespace bx;

namespace {

void put_msg(char *msg, int msglen, const std::string &s) {
  if (msg && msglen > 0) std::snprintf(msg, static_cast<size_t>(msglen), "%s", s.c_str());
}

std::string fmt(const char *f, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, f);
  std::vsnprintf(buf, sizeof buf, f, ap);
  va_end(ap);
  return buf;
}

#define BX_CUDA(call, msg, msglen)                                                    \
  do {                                                                                \
    cudaError_t e_ = (call);                                                          \
    if (e_ != cudaSuccess) {                                                          \
      put_msg(msg, msglen, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call); \
      return BX_RUNTIME;                                                              \
    }                                                                                 \
  } while (0)

constexpr int kMaxRosterList = 96;   // m-ETF / m-SCT
constexpr int kMaxRosterTopo = 1000; // m-TOPO

struct Fill {  // one k_fill range: byte i = byte (i mod 4) of the little-endian word
  void *ptr;
  uint32_t word;
  size_t bytes;
};

}  // namespace

struct bx_plan {
  int device = 0;
  bx_plan_options opt{0, -1, 0, 0, 0, -1, 0};
  int ngraphs = 0, njobs = 0, nprep = 0;
  std::vector<bx_graph> hg;
  std::vector<bx_job> hj;
  std::vector<DGraph> dg;
  std::vector<DPrep> dp;
  std::vector<DJob> dj;
  std::vector<int> prep_first;      // prep index -> 1 if first prep of its graph
  int max_ev = 0;                   // largest max(V, E) over graphs (prep grid)
  int total_V = 0;                  // need arrays of all graphs, concatenated (one segmented sort)
  int64_t *need_all = nullptr, *need_keys_all = nullptr;
  int32_t *iota_all = nullptr, *need_order_all = nullptr, *seg_off = nullptr;
  FillChunk *fill_dev = nullptr;    // per-step fills as k_fill chunks
  int nfill = 0;
  FillChunk *sim_fill_dev = nullptr;
  int nsim_fill = 0;
  std::vector<int> host_status;     // per job host-side validation result
  std::vector<std::string> host_msg;
  void *pool = nullptr;
  size_t pool_bytes = 0;
  DGraph *dg_dev = nullptr;
  DPrep *dp_dev = nullptr;
  DJob *dj_dev = nullptr;
  int32_t *order_dev = nullptr;     // launch lists: small | big parallel | big sequential
  int n_small = 0, n_etf = 0, n_bpar = 0, n_bseq = 0;  // n_etf: leading parallel m-ETF small jobs
  int n_sf[5] = {0, 0, 0, 0, 0};    // small-frontier (K2s) jobs, launched first: m-ETF, m-SCT with
                                    // shared-memory node state, then both with global node state;
                                    // [4]: sequential-comm m-ETF (K2q, seqsmall.cu)
  size_t sq_smem = 0;               // K2q shared memory (largest slot table among its jobs)
  size_t sf_smem[2] = {0, 0};
  std::vector<char> sf_global;      // job -> K2s with global node state
  std::vector<char> sf_seq;         // job -> K2q (sequential comm, small frontier)
  size_t topo_smem = 0;  // m-TOPO CTA: bitsets (+ counters) of the largest m-TOPO graph
  int32_t *sf_order_dev = nullptr;
  std::vector<char> prep_small;     // prep index -> K2s extras needed
  std::vector<int> job_kernel;      // BX_KERNEL_* of the general kernel each job is queued on
  cudaStream_t s2 = nullptr;        // big problems run beside the small ones
  cudaEvent_t fork = nullptr, join = nullptr;
  int32_t **queues_dev = nullptr;
  void *sort_tmp = nullptr;
  size_t sort_tmp_bytes = 0;
  std::vector<HostCopy> uploads;     // graph arrays: straight from the caller
  struct Staged {
    size_t off;
    const void *src;
    size_t bytes;
  };
  std::vector<Staged> staged;        // job inputs: packed into host_in, one copy
  struct OOff {
    size_t dev, start, eo, eoff, stats, err;
  };
  struct IOff {
    size_t cap, fav;
  };
  std::vector<OOff> out_off;
  std::vector<IOff> in_off;
  size_t in_bytes = 0, out_bytes = 0;
  char *dev_in = nullptr, *dev_out = nullptr;  // regions inside pool
  void *host_in = nullptr, *host_out = nullptr;  // pinned mirrors
  std::vector<int32_t> res_status;   // decoded by the last download
  std::vector<std::string> res_msg;
  std::vector<Fill> fills;
  int maxn = 1;      // largest roster among jobs that reach a placer kernel
  int maxn_all = 1;  // largest roster of any job (the simulator takes external placements)
  int64_t max_vn = 0;               // largest V*n over list-placer jobs
  bool any_topo = false, any_list = false;
  int launches = 0;
  cudaEvent_t ev[2] = {nullptr, nullptr};  // brackets the placer kernel(s) (ring slot 0)
  // per-step placer-kernel event pairs of the last kRing bx_plan_place calls
  // (owned plans; a borrowed one-shot plan keeps the single pair above)
  static constexpr int kRing = 64;
  std::vector<cudaEvent_t> ring0, ring1;
  int64_t places = 0;
  int64_t *prof = nullptr;                 // per-job latency breakdown (BX_PROFILE=1)
  // simulator
  void *sim_pool = nullptr;
  DSim *ds_dev = nullptr;
  std::vector<DSim> ds;
  std::vector<Fill> sim_fills;
  int sim_mem_mode = -1;
  // external placements (bx_simulate)
  bool external = false;
  // one-shot plans borrow pools, pinned mirrors, streams and events from
  // the calling thread's arena (arena.hpp) instead of owning them
  bool borrowed = false;
};

namespace bx {
Arena &thread_arena() {
  static thread_local std::vector<Arena *> per_device;
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) {
    cudaGetLastError();
    d = 0;
  }
  if (static_cast<int>(per_device.size()) <= d) per_device.resize(static_cast<size_t>(d) + 1, nullptr);
  if (!per_device[d]) per_device[d] = new Arena();
  return *per_device[d];
}
}  // namespace bx

static thread_local std::string g_last_error;

// Records the first pending CUDA launch error (kernel config, smem, ...).
static int launch_status() {
  cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return BX_OK;
  g_last_error = std::string("CUDA launch error: ") + cudaGetErrorString(e);
  return BX_RUNTIME;
}

extern "C" {

const char *bx_version(void) { return "baechi-b200 0.1 (sm_100a)"; }

const char *bx_last_error(void) { return g_last_error.c_str(); }

// Full text of the last one-shot call's error (msg[256] keeps a prefix).
static thread_local std::string g_last_message;
const char *bx_last_message(void) { return g_last_message.c_str(); }

int bx_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int bx_comm_time(const bx_comm *cm, int64_t bytes, int64_t *out_us) {
  if (bytes < 0) return BX_VALIDATION;
  *out_us = comm_time_exact(cm->intercept_us, cm->us_per_byte, bytes);
  return BX_OK;
}

int bx_build_adjacency(int32_t V, int32_t E, const int32_t *esrc, const int32_t *edst, int32_t *in_off,
                       int32_t *in_edge, int32_t *out_off, char *msg, int msglen) {
  for (int v = 0; v <= V; ++v) in_off[v] = out_off[v] = 0;
  for (int e = 0; e < E; ++e) {
    if (esrc[e] < 0 || esrc[e] >= V || edst[e] < 0 || edst[e] >= V) {
      put_msg(msg, msglen, fmt("meta edge %d references an unknown node", e));
      return BX_VALIDATION;
    }
    if (e > 0 && (esrc[e] < esrc[e - 1] || (esrc[e] == esrc[e - 1] && edst[e] <= edst[e - 1]))) {
      put_msg(msg, msglen, "meta edges must be sorted by (src, dst) and unique");
      return BX_VALIDATION;
    }
    in_off[edst[e] + 1]++;
    out_off[esrc[e] + 1]++;
  }
  for (int v = 0; v < V; ++v) {
    in_off[v + 1] += in_off[v];
    out_off[v + 1] += out_off[v];
  }
  std::vector<int32_t> pos(in_off, in_off + V);
  for (int e = 0; e < E; ++e) in_edge[pos[edst[e]]++] = e;
  put_msg(msg, msglen, "");
  return BX_OK;
}

void bx_plan_destroy(bx_plan *plan) {
  if (!plan) return;
  cudaSetDevice(plan->device);
  if (plan->borrowed) {  // pools, tables, streams and events belong to the thread's arena
    if (plan->prof) cudaFree(plan->prof);
    delete plan;
    return;
  }
  if (plan->pool) cudaFree(plan->pool);
  if (plan->host_in) cudaFreeHost(plan->host_in);
  if (plan->host_out) cudaFreeHost(plan->host_out);
  if (plan->sim_pool) cudaFree(plan->sim_pool);
  if (plan->sort_tmp) cudaFree(plan->sort_tmp);
  if (plan->prof) cudaFree(plan->prof);
  if (plan->fill_dev) cudaFree(plan->fill_dev);
  if (plan->sim_fill_dev) cudaFree(plan->sim_fill_dev);
  if (plan->ev[0]) cudaEventDestroy(plan->ev[0]);
  if (plan->ev[1]) cudaEventDestroy(plan->ev[1]);
  for (size_t i = 1; i < plan->ring0.size(); ++i) {
    cudaEventDestroy(plan->ring0[i]);
    cudaEventDestroy(plan->ring1[i]);
  }
  if (plan->fork) cudaEventDestroy(plan->fork);
  if (plan->join) cudaEventDestroy(plan->join);
  if (plan->s2) cudaStreamDestroy(plan->s2);
  delete plan;
}

int bx_plan_create(int32_t ngraphs, const bx_graph *graphs, int32_t njobs, const bx_job *jobs, int32_t device,
                   bx_plan **out, char *msg, int msglen) {
  return bx_plan_create_ex(ngraphs, graphs, njobs, jobs, device, nullptr, out, msg, msglen);
}

}  // extern "C"

namespace {
// Splits fills into k_fill chunks and uploads the table: to the arena slot
// `slot` for borrowed plans (left unowned), else to a fresh allocation.
int upload_fills(const std::vector<Fill> &fills, Arena *A, int slot, FillChunk **dev, int *n, char *msg,
                 int msglen) {
  std::vector<FillChunk> t;
  for (const Fill &f : fills) {
    for (size_t o = 0; o < f.bytes; o += kFillChunk) {
      const size_t b = std::min(kFillChunk, f.bytes - o);
      t.push_back({static_cast<char *>(f.ptr) + o, static_cast<uint32_t>(b), f.word});
    }
  }
  *n = static_cast<int>(t.size());
  if (t.empty()) return BX_OK;
  const size_t bytes = sizeof(FillChunk) * t.size();
  if (A) {
    char *pp = nullptr;
    BX_CUDA(A->device(bytes, &pp, slot), msg, msglen);
    *dev = nullptr;  // not owned
    BX_CUDA(cudaMemcpy(pp, t.data(), bytes, cudaMemcpyHostToDevice), msg, msglen);
    *dev = reinterpret_cast<FillChunk *>(pp);
    return BX_OK;
  }
  BX_CUDA(cudaMalloc(reinterpret_cast<void **>(dev), bytes), msg, msglen);
  BX_CUDA(cudaMemcpy(*dev, t.data(), bytes, cudaMemcpyHostToDevice), msg, msglen);
  return BX_OK;
}

// Frees a half-built plan on every early return of plan_create.
struct PlanGuard {
  bx_plan *p = nullptr;
  ~PlanGuard() {
    if (p) bx_plan_destroy(p);
  }
};
}  // namespace

static int plan_create(int32_t ngraphs, const bx_graph *graphs, int32_t njobs, const bx_job *jobs, int32_t device,
                       const bx_plan_options *options, bool borrow, bx_plan **out, char *msg, int msglen) {
  *out = nullptr;
  int ndev = bx_device_count();
  if (ndev <= 0) {
    put_msg(msg, msglen, "no CUDA device: the B200 placement engine has no CPU fallback");
    return BX_RUNTIME;
  }
  if (device < 0 || device >= ndev) {
    put_msg(msg, msglen, fmt("CUDA device %d out of range (%d visible)", device, ndev));
    return BX_RUNTIME;
  }
  BX_CUDA(cudaSetDevice(device), msg, msglen);
  auto *P = new (std::nothrow) bx_plan();
  if (!P) return BX_RUNTIME;
  PlanGuard guard;
  guard.p = P;
  P->device = device;
  P->borrowed = borrow;
  Arena *A = borrow ? &thread_arena() : nullptr;
  if (options) P->opt = *options;
  P->ngraphs = ngraphs;
  P->njobs = njobs;
  P->hg.assign(graphs, graphs + ngraphs);
  P->hj.assign(jobs, jobs + njobs);
  P->host_status.assign(njobs, 0);
  P->host_msg.assign(njobs, "");

  // prepared graphs: one per distinct (graph, intercept, per_byte)
  std::map<std::tuple<int, double, double>, int> prep_of;
  std::vector<int> job_prep(njobs);
  for (int i = 0; i < njobs; ++i) {
    const bx_job &J = jobs[i];
    if (J.graph < 0 || J.graph >= ngraphs) {
      put_msg(msg, msglen, fmt("job %d names graph %d of %d", i, J.graph, ngraphs));
      return BX_VALIDATION;
    }
    auto key = std::make_tuple(J.graph, J.cm.intercept_us, J.cm.us_per_byte);
    auto it = prep_of.find(key);
    if (it == prep_of.end()) it = prep_of.emplace(key, static_cast<int>(prep_of.size())).first;
    job_prep[i] = it->second;
    P->maxn_all = std::max(P->maxn_all, J.n);
  }
  P->nprep = static_cast<int>(prep_of.size());

  Layout L;
  struct GOff {
    size_t k, temp, perm, outb, esrc, edst, ebytes, in_off, in_edge, out_off, need, need_order, iota, need_keys,
        in_src, inpos, indeg_left, flags, queue, ksum;
  };
  std::vector<GOff> go(ngraphs);
  size_t max_sort_V = 0;
  for (int g = 0; g < ngraphs; ++g) {
    const bx_graph &G = graphs[g];
    GOff &o = go[g];
    o.k = L.take<int64_t>(G.V);
    o.temp = L.take<int64_t>(G.V);
    o.perm = L.take<int64_t>(G.V);
    o.outb = L.take<int64_t>(G.V);
    o.esrc = L.take<int32_t>(G.E);
    o.edst = L.take<int32_t>(G.E);
    o.ebytes = L.take<int64_t>(G.E);
    o.in_off = L.take<int32_t>(G.V + 1);
    o.in_edge = L.take<int32_t>(G.E);
    o.out_off = L.take<int32_t>(G.V + 1);
    o.need = o.need_order = o.iota = o.need_keys = static_cast<size_t>(P->total_V);  // element offsets
    P->total_V += G.V;
    o.in_src = L.take<int32_t>(G.E);
    o.inpos = L.take<int32_t>(G.E);
    o.indeg_left = L.take<int32_t>(G.V);
    o.flags = L.take<int32_t>(4);
    o.ksum = L.take<int64_t>(1);
    o.queue = L.take<int32_t>(2 * static_cast<size_t>(G.V));
    max_sort_V = std::max(max_sort_V, static_cast<size_t>(G.V));
    P->max_ev = std::max(P->max_ev, std::max(G.V, G.E));
  }
  const size_t need_at = L.take<int64_t>(P->total_V), need_keys_at = L.take<int64_t>(P->total_V);
  const size_t iota_at = L.take<int32_t>(P->total_V), need_order_at = L.take<int32_t>(P->total_V);
  const size_t seg_at = L.take<int32_t>(size_t(ngraphs) + 1);
  std::vector<std::pair<size_t, size_t>> po(P->nprep);  // in_c, cmax
  struct POff {
    size_t c32, nu, cnt, npk, ipk;
  };
  std::vector<POff> pso(P->nprep);
  std::vector<int> prep_graph(P->nprep);
  std::vector<std::pair<double, double>> prep_cm(P->nprep);
  for (auto &kv : prep_of) {
    int pi = kv.second;
    int g = std::get<0>(kv.first);
    prep_graph[pi] = g;
    prep_cm[pi] = {std::get<1>(kv.first), std::get<2>(kv.first)};
    po[pi].first = L.take<int64_t>(graphs[g].E);
    po[pi].second = L.take<int64_t>(1);
    pso[pi].c32 = L.take<int32_t>(graphs[g].E);
    pso[pi].nu = L.take<int32_t>(graphs[g].V);
    pso[pi].cnt = L.take<int32_t>(2);
    // K2s runs only in plans of at most 148 list jobs (`few` below)
    const bool few_jobs = std::count_if(jobs, jobs + njobs, [](const bx_job &J) { return J.algo != BX_ALGO_MTOPO; }) <= 148;
    pso[pi].npk = L.take<int4>(few_jobs ? size_t(graphs[g].V) : 1);
    pso[pi].ipk = L.take<uint2>(few_jobs ? graphs[g].E : 1);
  }
  struct JOff {
    size_t cap, fav, K, cache, dead, pending, alive, ready, rpos, cseq, nc, finish, urgent, scv, scg, pdev, pfin, K2, urgent2, ready2, alive2, ncw, newl, device_of,
        start, exec_order, exec_off, stats, err, sdone;
  };
  // Few large list-placer problems run the CTA-wide kernels (one problem per
  // CTA); many run one warp each. Decided here because the round kernel
  // needs double-buffered slot arrays. A job is "big" (CTA-wide kernels) when
  // V*n >= 2^17, or >= 2^15 in a plan of at most 148 list jobs; at most 120
  // big jobs (the largest), so the small ones keep SMs to run on.
  std::vector<int32_t> list_ids;
  for (int i = 0; i < njobs; ++i)
    if (jobs[i].algo != BX_ALGO_MTOPO) list_ids.push_back(i);
  auto vn = [&](int i) { return int64_t(graphs[jobs[i].graph].V) * std::max(jobs[i].n, 1); };
  std::stable_sort(list_ids.begin(), list_ids.end(), [&](int a, int b) { return vn(a) > vn(b); });
  // A plan of at most 148 list jobs gives every parallel-mode job its own
  // round-kernel CTA (faster per commit at every size measured,
  // profiles/r01c_kr_sweep.txt); sequential-mode jobs go wide from 2^15.
  // In a many-job sweep parallel-mode jobs all stay on the warp kernel: a
  // round CTA holds a whole SM's register file, and the sweep ran 14.0k
  // placements/s with none of them vs 13.2k with the 120 largest
  // (profiles/r01d_seq_policy.txt).
  const bool few = list_ids.size() <= 148;
  int64_t big_min = few ? (int64_t(1) << 15) : (int64_t(1) << 17);
  int64_t big_min_par = few ? 0 : INT64_MAX;
  if (P->opt.wide_min_vn >= 0) big_min = big_min_par = P->opt.wide_min_vn;
  std::vector<char> big(njobs, 0);
  size_t big_max = 120;
  if (P->opt.wide_max_jobs > 0) big_max = static_cast<size_t>(P->opt.wide_max_jobs);
  for (size_t r = 0; r < list_ids.size() && r < big_max; ++r) {
    const int i = list_ids[r];
    // small m-SCT problems commit one pair at a time more often (lifted
    // reservations dirty columns), where the lone warp beats the round CTA
    // (C3: 6.2 vs 7.2 ms); so they go wide only from 2^15 like sequential jobs
    const bool sct = jobs[i].algo == BX_ALGO_MSCT && jobs[i].fav_child != nullptr;
    if (vn(i) >= (jobs[i].cm.mode == BX_COMM_SEQUENTIAL || sct ? big_min : big_min_par)) big[i] = 1;
  }
  // job inputs (capacities, favourites) and outputs live in two contiguous
  // regions so an end-to-end step moves them with one copy each way, through
  // pinned host mirrors
  Layout LI, LO;
  LI.align = LO.align = 8;
  std::vector<JOff> jo(njobs);
  for (int i = 0; i < njobs; ++i) {
    const bx_job &J = jobs[i];
    const int64_t V = graphs[J.graph].V;
    const int64_t n = std::max(J.n, 1);
    JOff &o = jo[i];
    o.cap = LI.take<int64_t>(n);
    o.fav = LI.take<int32_t>(J.algo == BX_ALGO_MSCT && J.fav_child ? V : 1);
    o.K = L.take<int64_t>(V * n);
    o.cache = L.take<int64_t>(V * n);
    o.dead = L.take<uint8_t>(J.algo == BX_ALGO_MTOPO ? V * n : 1);  // m-TOPO's bitset scratch past shared memory
    o.pending = L.take<int32_t>(V);
    o.alive = L.take<int32_t>(V);
    o.ready = L.take<int32_t>(V);
    o.rpos = L.take<int32_t>(V);
    o.cseq = L.take<int32_t>(V);
    o.nc = L.take<int32_t>(V);
    o.finish = L.take<int64_t>(V);
    o.urgent = L.take<int64_t>(V);
    o.scv = L.take<int64_t>(256 * n);  // per lane of up to 8 warps
    o.scg = L.take<int32_t>(256 * n);
    o.pdev = L.take<int32_t>(graphs[J.graph].E);
    {
      const bool wide_plan = big[i] != 0;
      const int64_t Vr = wide_plan ? V : 1;
      o.K2 = L.take<int64_t>(Vr * (wide_plan ? n : 1));
      o.urgent2 = L.take<int64_t>(Vr);
      o.ready2 = L.take<int32_t>(Vr);
      o.alive2 = L.take<int32_t>(Vr);
      o.ncw = L.take<int32_t>(Vr);
      o.newl = L.take<int32_t>(Vr);
    }
    o.pfin = L.take<int64_t>(graphs[J.graph].E);
    o.sdone = L.take<int32_t>(1);
    o.stats = LO.take<int64_t>(3);
    o.err = LO.take<DErr>(1);
    o.start = LO.take<int64_t>(V);
    o.device_of = LO.take<int32_t>(V);
    o.exec_order = LO.take<int32_t>(V);
    o.exec_off = LO.take<int32_t>(n + 1);
  }
  size_t tables = L.take<DGraph>(ngraphs);
  size_t ptables = L.take<DPrep>(P->nprep);
  size_t jtables = L.take<DJob>(njobs);
  size_t qtables = L.take<int32_t *>(ngraphs);
  size_t otable = L.take<int32_t>(3 * size_t(njobs) + 3);
  size_t sftable = L.take<int32_t>(size_t(njobs) + 1);
  const size_t in_at = L.take<char>(LI.off), out_at = L.take<char>(LO.off);
  P->in_bytes = LI.off;
  P->out_bytes = LO.off;
  P->pool_bytes = L.off;
  cudaError_t ce;
  if (A) {
    char *pp = nullptr;
    ce = A->device(P->pool_bytes, &pp, 1);
    P->pool = pp;
    if (ce == cudaSuccess) ce = A->pinned(std::max<size_t>(P->in_bytes, 8), &P->host_in, 0);
    if (ce == cudaSuccess) ce = A->pinned(std::max<size_t>(P->out_bytes, 8), &P->host_out, 1);
  } else {
    ce = cudaMalloc(&P->pool, P->pool_bytes);
    if (ce == cudaSuccess) ce = cudaHostAlloc(&P->host_in, std::max<size_t>(P->in_bytes, 8), cudaHostAllocDefault);
    if (ce == cudaSuccess) ce = cudaHostAlloc(&P->host_out, std::max<size_t>(P->out_bytes, 8), cudaHostAllocDefault);
  }
  if (ce != cudaSuccess) {
    put_msg(msg, msglen, fmt("cudaMalloc of %zu bytes failed: %s", P->pool_bytes, cudaGetErrorString(ce)));
    return BX_RUNTIME;
  }
  void *pool = P->pool;
  P->dev_in = at<char>(pool, in_at);
  P->dev_out = at<char>(pool, out_at);
  // alignment gaps of the output region are copied by every download: give
  // them a defined value once
  BX_CUDA(cudaMemset(P->dev_out, 0, std::max<size_t>(P->out_bytes, 1)), msg, msglen);

  P->need_all = at<int64_t>(pool, need_at);
  P->need_keys_all = at<int64_t>(pool, need_keys_at);
  P->iota_all = at<int32_t>(pool, iota_at);
  P->need_order_all = at<int32_t>(pool, need_order_at);
  P->seg_off = at<int32_t>(pool, seg_at);
  {
    std::vector<int32_t> seg(static_cast<size_t>(ngraphs) + 1, 0);
    for (int g = 0; g < ngraphs; ++g) seg[g + 1] = seg[g] + graphs[g].V;
    BX_CUDA(cudaMemcpy(P->seg_off, seg.data(), 4 * seg.size(), cudaMemcpyHostToDevice), msg, msglen);
  }
  P->dg.resize(ngraphs);
  std::vector<int32_t *> queues(ngraphs);
  for (int g = 0; g < ngraphs; ++g) {
    const bx_graph &G = graphs[g];
    const GOff &o = go[g];
    DGraph &d = P->dg[g];
    d.V = G.V;
    d.E = G.E;
    d.k = at<int64_t>(pool, o.k);
    d.temp = at<int64_t>(pool, o.temp);
    d.perm = at<int64_t>(pool, o.perm);
    d.outb = at<int64_t>(pool, o.outb);
    d.esrc = at<int32_t>(pool, o.esrc);
    d.edst = at<int32_t>(pool, o.edst);
    d.ebytes = at<int64_t>(pool, o.ebytes);
    d.in_off = at<int32_t>(pool, o.in_off);
    d.in_edge = at<int32_t>(pool, o.in_edge);
    d.out_off = at<int32_t>(pool, o.out_off);
    d.need = at<int64_t>(pool, need_at) + o.need;
    d.need_order = at<int32_t>(pool, need_order_at) + o.need_order;
    d.iota = at<int32_t>(pool, iota_at) + o.iota;
    d.need_keys = at<int64_t>(pool, need_keys_at) + o.need_keys;
    d.in_src = at<int32_t>(pool, o.in_src);
    d.inpos = at<int32_t>(pool, o.inpos);
    d.indeg_left = at<int32_t>(pool, o.indeg_left);
    d.flags = at<int32_t>(pool, o.flags);
    d.ksum = at<int64_t>(pool, o.ksum);
    P->fills.push_back({d.ksum, 0, 8});
    queues[g] = at<int32_t>(pool, o.queue);
    auto up = [&](const void *dev, const void *host, size_t bytes) {
      if (bytes) P->uploads.push_back({const_cast<void *>(dev), host, bytes});
    };
    up(d.k, G.compute_us, 8 * size_t(G.V));
    up(d.temp, G.temp_bytes, 8 * size_t(G.V));
    up(d.perm, G.perm_bytes, 8 * size_t(G.V));
    up(d.outb, G.out_bytes, 8 * size_t(G.V));
    up(d.esrc, G.esrc, 4 * size_t(G.E));
    up(d.edst, G.edst, 4 * size_t(G.E));
    up(d.ebytes, G.tensor_bytes, 8 * size_t(G.E));
    up(d.in_off, G.in_off, 4 * size_t(G.V + 1));
    up(d.in_edge, G.in_edge, 4 * size_t(G.E));
    up(d.out_off, G.out_off, 4 * size_t(G.V + 1));
    P->fills.push_back({d.flags, 0, 16});
  }
  P->dp.resize(P->nprep);
  P->prep_first.assign(P->nprep, 0);
  std::vector<char> graph_seen(ngraphs, 0);
  for (int pi = 0; pi < P->nprep; ++pi) {
    DPrep &d = P->dp[pi];
    d.graph = prep_graph[pi];
    d.ic = prep_cm[pi].first;
    d.pb = prep_cm[pi].second;
    d.in_c = at<int64_t>(pool, po[pi].first);
    d.cmax = at<int64_t>(pool, po[pi].second);
    P->fills.push_back({d.cmax, 0, 8});
    d.in_c32 = at<int32_t>(pool, pso[pi].c32);
    d.nu = at<int32_t>(pool, pso[pi].nu);
    d.nu_count = at<int32_t>(pool, pso[pi].cnt);
    d.cbad = d.nu_count + 1;
    d.node_pack = at<int4>(pool, pso[pi].npk);
    d.in_pack = at<uint2>(pool, pso[pi].ipk);
    d.first = 0;
    if (!graph_seen[d.graph]) {
      graph_seen[d.graph] = 1;
      P->prep_first[pi] = 1;
      d.first = 1;
    }
  }
  // small-frontier kernel (K2s, smallsched.cu) eligibility inputs per graph:
  // largest in-degree and the producers whose out-edges carry different byte
  // counts (an upper bound of those with different comm times)
  std::vector<int> g_maxin(ngraphs, 0), g_nu(ngraphs, 0);
  for (int g = 0; g < ngraphs; ++g) {
    const bx_graph &G = graphs[g];
    for (int v = 0; v < G.V; ++v) g_maxin[g] = std::max(g_maxin[g], G.in_off[v + 1] - G.in_off[v]);
    for (int v = 0; v < G.V; ++v) {
      const int b = G.out_off[v], e = G.out_off[v + 1];
      for (int y = b + 1; y < e; ++y)
        if (G.tensor_bytes[y] != G.tensor_bytes[b]) {
          ++g_nu[g];
          break;
        }
    }
  }
  P->prep_small.assign(P->nprep, 0);
  P->sf_global.assign(njobs, 0);
  P->sf_seq.assign(njobs, 0);
  P->dj.resize(njobs);
  if (P->opt.profile == 1) {
    BX_CUDA(cudaMalloc(&P->prof, sizeof(int64_t) * kProfSlots * size_t(njobs)), msg, msglen);
    BX_CUDA(cudaMemset(P->prof, 0, sizeof(int64_t) * kProfSlots * size_t(njobs)), msg, msglen);
  }
  for (int i = 0; i < njobs; ++i) {
    const bx_job &J = jobs[i];
    const bx_graph &G = graphs[J.graph];
    const JOff &o = jo[i];
    DJob &d = P->dj[i];
    const int64_t V = G.V, n = std::max(J.n, 1);
    d.graph = J.graph;
    d.prep = job_prep[i];
    d.algo = J.algo;
    d.n = J.n;
    d.mode = J.cm.mode == BX_COMM_PARALLEL ? 1 : 0;
    d.skip = 0;
    d.cap = reinterpret_cast<int64_t *>(P->dev_in + o.cap);
    d.fav = nullptr;
    d.K = at<int64_t>(pool, o.K);
    d.cache = at<int64_t>(pool, o.cache);
    d.dead = at<uint8_t>(pool, o.dead);
    d.pending = at<int32_t>(pool, o.pending);
    d.alive = at<int32_t>(pool, o.alive);
    d.ready = at<int32_t>(pool, o.ready);
    d.rpos = at<int32_t>(pool, o.rpos);
    d.cseq = at<int32_t>(pool, o.cseq);
    d.nc = at<int32_t>(pool, o.nc);
    d.finish = at<int64_t>(pool, o.finish);
    d.urgent = at<int64_t>(pool, o.urgent);
    d.sc_val = at<int64_t>(pool, o.scv);
    d.sc_gen = at<int32_t>(pool, o.scg);
    d.pdev = at<int32_t>(pool, o.pdev);
    d.K2 = at<int64_t>(pool, o.K2);
    d.urgent2 = at<int64_t>(pool, o.urgent2);
    d.ready2 = at<int32_t>(pool, o.ready2);
    d.alive2 = at<int32_t>(pool, o.alive2);
    d.ncw = at<int32_t>(pool, o.ncw);
    d.newl = at<int32_t>(pool, o.newl);
    d.pfin = at<int64_t>(pool, o.pfin);
    d.device_of = reinterpret_cast<int32_t *>(P->dev_out + o.device_of);
    d.start = reinterpret_cast<int64_t *>(P->dev_out + o.start);
    d.exec_order = reinterpret_cast<int32_t *>(P->dev_out + o.exec_order);
    d.exec_off = reinterpret_cast<int32_t *>(P->dev_out + o.exec_off);
    d.stats = reinterpret_cast<int64_t *>(P->dev_out + o.stats);
    d.err = reinterpret_cast<DErr *>(P->dev_out + o.err);
    P->out_off.push_back({o.device_of, o.start, o.exec_order, o.exec_off, o.stats, o.err});
    // a job that is never placed (host validation) or fails in the placer
    // leaves device_of = -1 and empty exec lists, so a later simulate of it
    // fails validation instead of walking stale lists
    P->fills.push_back({d.device_of, 0xffffffffu, 4 * size_t(V)});
    P->fills.push_back({d.exec_off, 0, 4 * size_t(n + 1)});
    P->in_off.push_back({o.cap, o.fav});
    d.prof = P->prof ? P->prof + static_cast<size_t>(kProfSlots) * i : nullptr;
    // host-side validation in the reference's order
    std::string why;
    int st = 0;
    if (J.algo == BX_ALGO_MSCT && J.fav_child && J.fav_len != 0 && J.fav_len != G.V) {
      st = BX_VALIDATION;
      why = "favorite map does not match graph size";  // placers.cpp:306-309
    } else if (J.n <= 0) {
      st = BX_VALIDATION;
      why = "device roster is empty";  // placers.cpp:20-22
    } else {
      for (int x = 0; x < J.n; ++x)
        if (J.capacity[x] <= 0) {
          st = BX_VALIDATION;
          why = "device capacities must be positive";  // placers.cpp:25-27
        }
    }
    if (J.algo < 0 || J.algo > 2) {
      st = BX_VALIDATION;
      why = "unknown placement algorithm";
    }
    // per-device scheduling state lives in shared memory (the round kernel's
    // 32-entry column lists: ~1.8 KB per device); larger rosters are refused
    // per job instead of failing every launch of the plan
    const int lim = J.algo == BX_ALGO_MTOPO ? kMaxRosterTopo : kMaxRosterList;
    if (st == 0 && J.n > lim) {
      st = BX_RUNTIME;
      why = fmt("a roster of %d devices exceeds this engine's limit of %d per problem", J.n, lim);
    }
    P->host_status[i] = st;
    P->host_msg[i] = why;
    d.skip = st != 0;
    if (J.n > 0) P->staged.push_back({P->in_off[i].cap, J.capacity, 8 * size_t(J.n)});
    if (!d.skip) {
      if (J.algo == BX_ALGO_MSCT && J.fav_child && J.fav_len == G.V && G.V > 0) {
        d.fav = reinterpret_cast<int32_t *>(P->dev_in + o.fav);
        P->staged.push_back({P->in_off[i].fav, J.fav_child, 4 * size_t(V)});
      }
      if (J.algo == BX_ALGO_MTOPO) {
        P->any_topo = true;
        P->topo_smem = std::max(P->topo_smem, topo_smem_bytes(G.V, 200 * 1024));
      } else {
        P->any_list = true;
        P->max_vn = std::max(P->max_vn, int64_t(G.V) * J.n);
      }
    }
    // parallel comm, every producer sends the same bytes on all its
    // out-edges: the list placers never touch the cache (DJob::nocache)
    d.nocache = J.algo != BX_ALGO_MTOPO && J.cm.mode == BX_COMM_PARALLEL && g_nu[J.graph] == 0;
    if (!d.nocache) P->fills.push_back({d.cache, 0xffffffffu, 8 * size_t(V * n)});
    if (d.skip) {  // the status record carries the host verdict (message kept host-side)
      P->fills.push_back({d.err, static_cast<uint32_t>(st), 4});
      P->fills.push_back({reinterpret_cast<char *>(d.err) + 4, static_cast<uint32_t>(E_HOST), 4});
      P->fills.push_back({reinterpret_cast<char *>(d.err) + 8, 0, sizeof(DErr) - 8});
    } else {
      P->fills.push_back({d.err, 0, sizeof(DErr)});
    }
    // K2s: parallel-comm list jobs of single-graph-sized plans whose per-node
    // state fits one SM's shared memory; the kernel re-checks the value
    // bounds on the device and leaves the job to the general kernels if any
    // fails (or its frontier outgrows 256 pairs)
    d.sdone = nullptr;
    d.nucap = g_nu[J.graph];
    d.maxin = g_maxin[J.graph];
    // (64 devices for m-ETF; the kernel takes more than 32 only without cache rows)
    if (!d.skip && few && J.algo != BX_ALGO_MTOPO && J.cm.mode == BX_COMM_PARALLEL &&
        J.n <= (J.algo == BX_ALGO_MSCT ? 32 : 64) && G.V > 0 &&
        G.V < (1 << 26) && !P->opt.no_small_frontier && P->opt.wide_min_vn < 0) {
      const int nccap = J.n * std::max(1, d.maxin);
      const size_t sm = small_smem_bytes_host(G.V, J.n, d.nucap, nccap);
      const size_t smg = small_smem_bytes_host(0, J.n, d.nucap, nccap);  // node state in HBM
      const bool glob = sm > 200 * 1024;
      if (!glob || smg <= 200 * 1024) {
        d.sdone = at<int32_t>(pool, o.sdone);
        P->fills.push_back({d.sdone, 0, 4});
        // (node state in HBM: + the pending counts as bytes when they fit)
        P->sf_smem[glob] = std::max(P->sf_smem[glob],
                                    glob ? smg + small_pend_bytes_host(G.V, J.n, d.nucap, nccap, d.maxin) : sm);
        P->sf_global[i] = glob;
        P->prep_small[job_prep[i]] = 1;
      }
    }
    // K2q: sequential-comm m-ETF jobs of single-graph-sized plans (the kernel
    // leaves the job to the general kernels once its frontier passes 512 pairs)
    if (!d.skip && few && J.algo != BX_ALGO_MTOPO && J.cm.mode != BX_COMM_PARALLEL && d.fav == nullptr &&
        J.n <= 32 && G.V > 0 && G.V < (1 << 26) && !P->opt.no_small_frontier && P->opt.wide_min_vn < 0) {
      d.sdone = at<int32_t>(pool, o.sdone);
      P->fills.push_back({d.sdone, 0, 4});
      P->sq_smem = std::max(P->sq_smem, seq_small_smem_bytes_host(J.n, G.V, d.maxin));
      P->sf_seq[i] = 1;
      P->prep_small[job_prep[i]] = 1;
    }
  }
  // shared-memory slices are sized by the largest roster among jobs that
  // reach a kernel: a rejected job's roster never costs the others a launch
  P->maxn = 1;
  for (int i = 0; i < njobs; ++i)
    if (!P->dj[i].skip) P->maxn = std::max(P->maxn, jobs[i].n);
  P->dg_dev = at<DGraph>(pool, tables);
  P->dp_dev = at<DPrep>(pool, ptables);
  P->dj_dev = at<DJob>(pool, jtables);
  P->queues_dev = at<int32_t *>(pool, qtables);
  P->order_dev = at<int32_t>(pool, otable);
  P->sf_order_dev = at<int32_t>(pool, sftable);
  {
    std::vector<int32_t> lists[5], all;
    for (int i = 0; i < njobs; ++i) {
      if (!P->dj[i].sdone) continue;
      if (P->sf_seq[i]) lists[4].push_back(i);
      else lists[2 * P->sf_global[i] + (P->dj[i].algo == BX_ALGO_MSCT && P->dj[i].fav ? 1 : 0)].push_back(i);
    }
    for (int k = 0; k < 5; ++k) {
      P->n_sf[k] = static_cast<int>(lists[k].size());
      all.insert(all.end(), lists[k].begin(), lists[k].end());
    }
    if (!all.empty())
      BX_CUDA(cudaMemcpy(P->sf_order_dev, all.data(), 4 * all.size(), cudaMemcpyHostToDevice), msg, msglen);
  }
  {
    // three launch lists, each longest-first: small (one warp per job),
    // big parallel-mode (round kernel), big sequential-mode (8-warp kernel)
    std::vector<int32_t> small, sgen, bpar, bseq;
    for (int i : list_ids) {
      if (P->dj[i].skip) continue;
      const bool etf = jobs[i].cm.mode == BX_COMM_PARALLEL && P->dj[i].fav == nullptr;
      if (!big[i]) (etf ? small : sgen).push_back(i);
      else if (jobs[i].cm.mode == BX_COMM_PARALLEL) bpar.push_back(i);
      else bseq.push_back(i);
    }
    P->job_kernel.assign(njobs, BX_KERNEL_NONE);
    for (int i = 0; i < njobs; ++i)
      if (!P->dj[i].skip && jobs[i].algo == BX_ALGO_MTOPO) P->job_kernel[i] = BX_KERNEL_MTOPO;
    for (int i : small) P->job_kernel[i] = BX_KERNEL_WARP;
    for (int i : sgen) P->job_kernel[i] = BX_KERNEL_WARP;
    for (int i : bpar) P->job_kernel[i] = BX_KERNEL_ROUNDS;
    for (int i : bseq) P->job_kernel[i] = BX_KERNEL_CTA_SEQ;
    P->n_etf = static_cast<int>(small.size());
    small.insert(small.end(), sgen.begin(), sgen.end());
    std::vector<int32_t> all(small);
    all.insert(all.end(), bpar.begin(), bpar.end());
    all.insert(all.end(), bseq.begin(), bseq.end());
    P->n_small = static_cast<int>(small.size());
    P->n_bpar = static_cast<int>(bpar.size());
    P->n_bseq = static_cast<int>(bseq.size());
    if (!all.empty())
      BX_CUDA(cudaMemcpy(P->order_dev, all.data(), 4 * all.size(), cudaMemcpyHostToDevice), msg, msglen);
  }
  if (A) {
    P->s2 = A->side_stream();
    P->fork = A->event(0, false);
    P->join = A->event(1, false);
  } else {
    BX_CUDA(cudaStreamCreateWithFlags(&P->s2, cudaStreamNonBlocking), msg, msglen);
    BX_CUDA(cudaEventCreateWithFlags(&P->fork, cudaEventDisableTiming), msg, msglen);
    BX_CUDA(cudaEventCreateWithFlags(&P->join, cudaEventDisableTiming), msg, msglen);
  }
  // descriptor tables are static: copy once
  BX_CUDA(cudaMemcpy(P->dg_dev, P->dg.data(), sizeof(DGraph) * ngraphs, cudaMemcpyHostToDevice), msg, msglen);
  BX_CUDA(cudaMemcpy(P->dp_dev, P->dp.data(), sizeof(DPrep) * P->nprep, cudaMemcpyHostToDevice), msg, msglen);
  BX_CUDA(cudaMemcpy(P->dj_dev, P->dj.data(), sizeof(DJob) * njobs, cudaMemcpyHostToDevice), msg, msglen);
  BX_CUDA(cudaMemcpy(P->queues_dev, queues.data(), sizeof(int32_t *) * ngraphs, cudaMemcpyHostToDevice), msg,
          msglen);
  // radix-sort scratch sized for the largest graph
  {
    (void)max_sort_V;
    size_t bytes = 0;
    sort_needs_all(nullptr, bytes, P->need_all, P->need_keys_all, P->iota_all, P->need_order_all, P->total_V, ngraphs,
                   P->seg_off, nullptr);
    P->sort_tmp_bytes = std::max<size_t>(bytes, 256);
    if (A) {
      char *pp = nullptr;
      BX_CUDA(A->device(P->sort_tmp_bytes, &pp, 3), msg, msglen);
      P->sort_tmp = pp;
    } else {
      BX_CUDA(cudaMalloc(&P->sort_tmp, P->sort_tmp_bytes), msg, msglen);
    }
  }
  if (A) {
    P->ev[0] = A->event(2, true);
    P->ev[1] = A->event(3, true);
  } else {
    BX_CUDA(cudaEventCreate(&P->ev[0]), msg, msglen);
    BX_CUDA(cudaEventCreate(&P->ev[1]), msg, msglen);
  }
  P->ring0.assign(1, P->ev[0]);
  P->ring1.assign(1, P->ev[1]);
  if (!A) {
    for (int i = 1; i < bx_plan::kRing; ++i) {
      cudaEvent_t a = nullptr, b = nullptr;
      BX_CUDA(cudaEventCreate(&a), msg, msglen);
      BX_CUDA(cudaEventCreate(&b), msg, msglen);
      P->ring0.push_back(a);
      P->ring1.push_back(b);
    }
  }
  {
    int rc = upload_fills(P->fills, A, 4, &P->fill_dev, &P->nfill, msg, msglen);
    if (rc) return rc;
  }
  guard.p = nullptr;
  *out = P;
  put_msg(msg, msglen, "");
  return BX_OK;
}

extern "C" {

int bx_plan_create_ex(int32_t ngraphs, const bx_graph *graphs, int32_t njobs, const bx_job *jobs, int32_t device,
                      const bx_plan_options *options, bx_plan **out, char *msg, int msglen) {
  return plan_create(ngraphs, graphs, njobs, jobs, device, options, false, out, msg, msglen);
}

int bx_plan_upload(bx_plan *P, void *stream) {
  cudaSetDevice(P->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  for (const HostCopy &c : P->uploads) {
    if (cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, s) != cudaSuccess) return BX_RUNTIME;
  }
  // the previous upload of host_in may still be in flight on this stream
  if (cudaStreamSynchronize(s) != cudaSuccess) return BX_RUNTIME;
  for (const auto &st : P->staged) std::memcpy(static_cast<char *>(P->host_in) + st.off, st.src, st.bytes);
  if (P->in_bytes &&
      cudaMemcpyAsync(P->dev_in, P->host_in, P->in_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return BX_RUNTIME;
  return BX_OK;
}

int bx_plan_place(bx_plan *P, void *stream) {
  cudaSetDevice(P->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  P->launches = 0;
  launch_fill(P->fill_dev, P->nfill, s);
  P->launches += P->nfill > 0;
  launch_prep_all(P->dg_dev, P->dp_dev, P->nprep, P->max_ev, s);
  P->launches += P->nprep > 0 && P->max_ev > 0;
  for (int pi = 0; pi < P->nprep; ++pi) {
    if (!P->prep_small[pi]) continue;
    const DGraph &g = P->dg[P->dp[pi].graph];
    cudaMemsetAsync(P->dp[pi].nu_count, 0, 8, s);
    launch_prep_small(g, P->dp[pi], s);
    P->launches += 2;
  }
  if (P->total_V > 0 && P->any_list) {  // need_order serves the list placers only
    size_t bytes = P->sort_tmp_bytes;
    cudaError_t e = sort_needs_all(P->sort_tmp, bytes, P->need_all, P->need_keys_all, P->iota_all, P->need_order_all,
                                   P->total_V, P->ngraphs, P->seg_off, s);
    if (e != cudaSuccess) {
      g_last_error = std::string("need sort: ") + cudaGetErrorString(e);
      return BX_RUNTIME;
    }
    P->launches += 3;
  }
  launch_kahn(P->dg_dev, P->queues_dev, P->ngraphs, s);
  P->launches += 1;
  const size_t slot = static_cast<size_t>(P->places % static_cast<int64_t>(P->ring0.size()));
  cudaEventRecord(P->ring0[slot], s);
  if (P->n_sf[0] + P->n_sf[1] + P->n_sf[2] + P->n_sf[3] > 0) {
    launch_small_frontier(P->dj_dev, P->sf_order_dev, P->n_sf, P->dg_dev, P->dp_dev, P->sf_smem,
                          P->prof != nullptr, s);
    for (int k = 0; k < 4; ++k) P->launches += P->n_sf[k] > 0;
  }
  if (P->n_sf[4] > 0) {
    launch_seq_small(P->dj_dev, P->sf_order_dev + P->n_sf[0] + P->n_sf[1] + P->n_sf[2] + P->n_sf[3], P->n_sf[4],
                     P->dg_dev, P->dp_dev, P->sq_smem, P->prof != nullptr, s);
    P->launches += 1;
  }
  const bool fork = (P->n_small > 0 && (P->n_bpar + P->n_bseq) > 0) || (P->n_etf > 0 && P->n_small > P->n_etf);
  cudaStream_t sb = fork ? P->s2 : s;
  if (fork) {
    cudaEventRecord(P->fork, s);
    cudaStreamWaitEvent(P->s2, P->fork, 0);
  }
  launch_placers(P->dj_dev, P->order_dev, P->n_small, P->n_etf, P->n_bpar, P->n_bseq, P->njobs, P->dg_dev,
                 P->dp_dev,
                 P->maxn, P->prof != nullptr, P->opt.list_len, s, sb);
  if (P->any_topo) launch_topo(P->dj_dev, P->njobs, P->dg_dev, P->dp_dev, P->topo_smem, s);
  if (fork) {
    cudaEventRecord(P->join, P->s2);
    cudaStreamWaitEvent(s, P->join, 0);
  }
  cudaEventRecord(P->ring1[slot], s);
  P->places++;
  P->launches += (P->any_topo ? 1 : 0) + (P->n_etf > 0) + (P->n_small > P->n_etf) + (P->n_bpar > 0) + (P->n_bseq > 0);
  return launch_status();
}

int bx_plan_launch_count(const bx_plan *P) { return P->launches; }

// The output region's device->host copy into the pinned mirror, enqueued on
// `stream` and not waited for (bx_plan_download waits and decodes).
int bx_plan_download_async(bx_plan *P, void *stream) {
  cudaSetDevice(P->device);
  if (P->out_bytes == 0) return BX_OK;
  return cudaMemcpyAsync(P->host_out, P->dev_out, P->out_bytes, cudaMemcpyDeviceToHost,
                         static_cast<cudaStream_t>(stream)) == cudaSuccess
             ? BX_OK
             : BX_RUNTIME;
}

int bx_plan_job_kernel(bx_plan *P, int32_t job) {
  if (job < 0 || job >= P->njobs) return BX_KERNEL_NONE;
  if (P->dj[job].sdone) {
    int32_t done = 0;
    cudaSetDevice(P->device);
    if (cudaMemcpy(&done, P->dj[job].sdone, 4, cudaMemcpyDeviceToHost) == cudaSuccess && done)
      return P->sf_seq[job] ? BX_KERNEL_SEQ_SMALL : BX_KERNEL_SMALL_FRONTIER;
  }
  return P->job_kernel[job];
}

int bx_plan_profile(bx_plan *P, int32_t job, int64_t *out16) {
  cudaSetDevice(P->device);
  if (!P->prof || job < 0 || job >= P->njobs) return BX_VALIDATION;
  if (cudaMemcpy(out16, P->prof + static_cast<size_t>(kProfSlots) * job, sizeof(int64_t) * kProfSlots,
                 cudaMemcpyDeviceToHost) != cudaSuccess)
    return BX_RUNTIME;
  return BX_OK;
}

float bx_plan_kernel_ms(bx_plan *P) {
  float ms = -1.0f;
  return bx_plan_kernel_times(P, 1, &ms) == 1 ? ms : -1.0f;
}

int bx_plan_kernel_times(bx_plan *P, int32_t count, float *ms) {
  cudaSetDevice(P->device);
  const int64_t ring = static_cast<int64_t>(P->ring0.size());
  const int64_t have = std::min<int64_t>({static_cast<int64_t>(count), P->places, ring});
  for (int64_t i = 0; i < have; ++i) {
    const int64_t step = P->places - have + i;
    const size_t slot = static_cast<size_t>(step % ring);
    if (cudaEventSynchronize(P->ring1[slot]) != cudaSuccess) return -1;
    if (cudaEventElapsedTime(&ms[i], P->ring0[slot], P->ring1[slot]) != cudaSuccess) return -1;
  }
  return static_cast<int>(have);
}

int bx_plan_output_region(const bx_plan *P, void **dev, int64_t *bytes) {
  *dev = P->dev_out;
  *bytes = static_cast<int64_t>(P->out_bytes);
  return BX_OK;
}

int bx_plan_job_outputs(const bx_plan *P, int32_t job, int64_t *offs6) {
  if (job < 0 || job >= P->njobs) return BX_VALIDATION;
  const auto &o = P->out_off[job];
  offs6[0] = static_cast<int64_t>(o.dev);
  offs6[1] = static_cast<int64_t>(o.start);
  offs6[2] = static_cast<int64_t>(o.eo);
  offs6[3] = static_cast<int64_t>(o.eoff);
  offs6[4] = static_cast<int64_t>(o.stats);
  offs6[5] = static_cast<int64_t>(o.err);
  return BX_OK;
}

static std::string cycle_message(const bx_plan *P, int g, cudaStream_t s) {
  const bx_graph &G = P->hg[g];
  std::vector<int32_t> left(G.V);
  cudaMemcpyAsync(left.data(), P->dg[g].indeg_left, 4 * size_t(G.V), cudaMemcpyDeviceToHost, s);
  cudaStreamSynchronize(s);
  std::string m = "meta graph is cyclic; groups of base node ids {";
  bool first = true;
  for (int i = 0; i < G.V; ++i) {
    if (left[i] > 0) {
      long long id = G.first_id ? static_cast<long long>(G.first_id[i]) : i;
      m += (first ? "" : ", ") + std::to_string(id);
      first = false;
    }
  }
  return m + "} remain";
}

// Device -> pinned host mirror (one copy), then per-job status decode; with
// `out` non-null the arrays are also copied into the caller's buffers.
int bx_plan_download(bx_plan *P, void *stream, bx_placement *out) {
  cudaSetDevice(P->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t ce = cudaSuccess;
  if (P->out_bytes) ce = cudaMemcpyAsync(P->host_out, P->dev_out, P->out_bytes, cudaMemcpyDeviceToHost, s);
  if (ce == cudaSuccess) ce = cudaStreamSynchronize(s);
  P->res_status.assign(P->njobs, 0);
  P->res_msg.assign(P->njobs, "");
  if (ce != cudaSuccess) {
    g_last_error = std::string("download: ") + cudaGetErrorString(ce);
    for (int i = 0; i < P->njobs; ++i) {
      P->res_status[i] = BX_RUNTIME;
      P->res_msg[i] = g_last_error;
      if (out) {
        out[i].status = BX_RUNTIME;
        put_msg(out[i].msg, sizeof out[i].msg, g_last_error);
      }
    }
    return BX_RUNTIME;
  }
  const char *H = static_cast<const char *>(P->host_out);
  for (int i = 0; i < P->njobs; ++i) {
    const DJob &d = P->dj[i];
    const bx_plan::OOff &o = P->out_off[i];
    int status;
    std::string m;
    if (d.skip) {
      status = P->host_status[i];
      m = P->host_msg[i];
    } else {
      const DErr &e = *reinterpret_cast<const DErr *>(H + o.err);
      status = e.status;
      switch (e.code) {
        case E_NONE:
          break;
        case E_FITS_NONE:
          m = "node " + std::to_string(e.a) + " fits on no device";
          break;
        case E_NO_PAIR:
          m = "no schedulable (node, device) pair remains";
          break;
        case E_CYCLE:
          m = cycle_message(P, d.graph, s);
          break;
        case E_NEG_BYTES:
          m = "comm_time: negative byte count";
          break;
        case E_TOPO_CAP:
          m = "m-topo per-device cap " + std::to_string(e.a) + " bytes exceeds the smallest device capacity " +
              std::to_string(e.b) + "; use m-etf or m-sct for tight memory limits";
          break;
        default:
          m = "internal error code " + std::to_string(e.code);
          status = BX_RUNTIME;
      }
    }
    P->res_status[i] = status;
    P->res_msg[i] = m;
    if (!out) continue;
    bx_placement &r = out[i];
    r.status = status;
    put_msg(r.msg, sizeof r.msg, m);
    const int64_t *st = reinterpret_cast<const int64_t *>(H + o.stats);
    for (int k = 0; k < 3; ++k) r.stats[k] = status == 0 && !d.skip ? st[k] : 0;
    if (status != 0 || d.skip) continue;
    const int V = P->hg[d.graph].V;
    if (r.device_of) std::memcpy(r.device_of, H + o.dev, 4 * size_t(V));
    if (r.start_us) std::memcpy(r.start_us, H + o.start, 8 * size_t(V));
    if (r.exec_order) std::memcpy(r.exec_order, H + o.eo, 4 * size_t(V));
    if (r.exec_off) std::memcpy(r.exec_off, H + o.eoff, 4 * size_t(d.n + 1));
  }
  return BX_OK;
}

// Zero-copy view of job `job`'s placement inside the plan's pinned host
// mirror (valid until the next bx_plan_download or bx_plan_destroy).
int64_t bx_plan_message(const bx_plan *P, int32_t job, char *buf, int64_t buflen) {
  if (job < 0 || job >= P->njobs || P->res_msg.empty()) return -1;
  const std::string &m = P->res_msg[job];
  if (buf && buflen > 0) {
    const size_t k = std::min(m.size(), static_cast<size_t>(buflen - 1));
    std::memcpy(buf, m.data(), k);
    buf[k] = 0;
  }
  return static_cast<int64_t>(m.size());
}

int bx_plan_result_view(bx_plan *P, int32_t job, bx_placement *view) {
  if (job < 0 || job >= P->njobs || P->res_status.empty()) return BX_VALIDATION;
  const bx_plan::OOff &o = P->out_off[job];
  char *H = static_cast<char *>(P->host_out);
  view->device_of = reinterpret_cast<int32_t *>(H + o.dev);
  view->start_us = reinterpret_cast<int64_t *>(H + o.start);
  view->exec_order = reinterpret_cast<int32_t *>(H + o.eo);
  view->exec_off = reinterpret_cast<int32_t *>(H + o.eoff);
  view->status = P->res_status[job];
  put_msg(view->msg, sizeof view->msg, P->res_msg[job]);
  const int64_t *st = reinterpret_cast<const int64_t *>(H + o.stats);
  for (int k = 0; k < 3; ++k) view->stats[k] = view->status == 0 && !P->dj[job].skip ? st[k] : 0;
  return BX_OK;
}

// ---- simulator -----------------------------------------------------------
static int sim_setup(bx_plan *P, char *msg, int msglen) {
  if (P->sim_pool) return BX_OK;
  Layout L;
  struct SOff {
    size_t mem, peak, xfree, qpos, busy, cl, fin, sq, res, sent, ht, hk, seen, db, dc, start, dev3n, xfer4, mk, err;
    size_t pos, psrc, cx, ffin, sx, bucket, mb, first, flow8, rcnt, rp_off, rp_src, rp_c, kx, dv, ninp, tr, trn;
  };
  std::vector<SOff> so(P->njobs);
  for (int i = 0; i < P->njobs; ++i) {
    const bx_graph &G = P->hg[P->dj[i].graph];
    const int64_t V = G.V, E = G.E, n = std::max(P->dj[i].n, 1);
    SOff &o = so[i];
    o.mem = L.take<int64_t>(n);
    o.peak = L.take<int64_t>(n);
    o.xfree = L.take<int64_t>(n);
    o.qpos = L.take<int32_t>(n);
    o.busy = L.take<uint8_t>(n);
    o.cl = L.take<int32_t>(V);
    o.fin = L.take<uint8_t>(V);
    o.sq = L.take<uint8_t>(V);
    o.res = L.take<uint8_t>(V * n);
    o.sent = L.take<uint8_t>(V * n);
    o.ht = L.take<int64_t>(2 * n + E + 16);
    o.hk = L.take<int64_t>(2 * n + E + 16);
    o.seen = L.take<int32_t>(V);
    o.db = L.take<int64_t>(n);
    o.dc = L.take<int32_t>(n);
    o.start = L.take<int64_t>(V);
    o.dev3n = L.take<int64_t>(3 * n);
    o.xfer4 = L.take<int64_t>(4);
    o.mk = L.take<int64_t>(1);
    o.err = L.take<DErr>(1);
    o.pos = L.take<int32_t>(V);
    o.psrc = L.take<int32_t>(E);
    o.cx = L.take<int64_t>(E);
    o.ffin = L.take<int64_t>(V);
    o.sx = L.take<int64_t>(V);
    o.bucket = L.take<int64_t>(V);
    o.mb = L.take<int64_t>(V * n);
    o.first = L.take<uint8_t>(E);
    o.flow8 = L.take<unsigned long long>(8);
    o.rcnt = L.take<int32_t>(V);
    o.rp_off = L.take<int32_t>(V + 1);
    o.rp_src = L.take<int32_t>(E);
    o.rp_c = L.take<int64_t>(E);
    o.kx = L.take<int64_t>(V);
    o.dv = L.take<int64_t>(4 * n);
    o.ninp = L.take<int32_t>(V);
    // every event is a start, a finish or one end of a transfer, and a
    // (producer, device) transfer needs a consumer edge: <= 2V + 2E events
    o.tr = P->opt.sim_trace ? L.take<int64_t>(4 * (2 * V + 2 * E + 4)) : 0;
    o.trn = L.take<unsigned long long>(1);
  }
  size_t tab = L.take<DSim>(P->njobs);
  if (P->borrowed) {
    char *pp = nullptr;
    BX_CUDA(thread_arena().device(L.off, &pp, 2), msg, msglen);
    P->sim_pool = pp;
  } else {
    BX_CUDA(cudaMalloc(&P->sim_pool, L.off), msg, msglen);
  }
  void *pool = P->sim_pool;
  P->ds.resize(P->njobs);
  for (int i = 0; i < P->njobs; ++i) {
    const DJob &j = P->dj[i];
    const bx_job &J = P->hj[i];
    const bx_graph &G = P->hg[j.graph];
    const SOff &o = so[i];
    DSim &d = P->ds[i];
    const int64_t V = G.V, E = G.E, n = std::max(j.n, 1);
    d.graph = j.graph;
    d.n = j.n;
    d.mode = j.mode;
    d.ic = J.cm.intercept_us;
    d.pb = J.cm.us_per_byte;
    d.cap = j.cap;
    d.device_of = j.device_of;
    d.exec_order = j.exec_order;
    d.exec_off = j.exec_off;
    d.mem = at<int64_t>(pool, o.mem);
    d.peak = at<int64_t>(pool, o.peak);
    d.xfree = at<int64_t>(pool, o.xfree);
    d.qpos = at<int32_t>(pool, o.qpos);
    d.busy = at<uint8_t>(pool, o.busy);
    d.consumers_left = at<int32_t>(pool, o.cl);
    d.finished = at<uint8_t>(pool, o.fin);
    d.start_q = at<uint8_t>(pool, o.sq);
    d.resident = at<uint8_t>(pool, o.res);
    d.sent = at<uint8_t>(pool, o.sent);
    d.heap_t = at<int64_t>(pool, o.ht);
    d.heap_k = at<int64_t>(pool, o.hk);
    d.heap_cap = 2 * n + E + 16;
    d.seen = at<int32_t>(pool, o.seen);
    d.dest_bytes = at<int64_t>(pool, o.db);
    d.dest_cnt = at<int32_t>(pool, o.dc);
    d.start = at<int64_t>(pool, o.start);
    d.dev3n = at<int64_t>(pool, o.dev3n);
    d.xfer4 = at<int64_t>(pool, o.xfer4);
    d.makespan = at<int64_t>(pool, o.mk);
    d.err = at<DErr>(pool, o.err);
    d.pos = at<int32_t>(pool, o.pos);
    d.psrc = at<int32_t>(pool, o.psrc);
    d.cx = at<int64_t>(pool, o.cx);
    d.fin = at<int64_t>(pool, o.ffin);
    d.sx = at<int64_t>(pool, o.sx);
    d.bucket = at<int64_t>(pool, o.bucket);
    d.mb = at<int64_t>(pool, o.mb);
    d.first = at<uint8_t>(pool, o.first);
    d.flow8 = at<unsigned long long>(pool, o.flow8);
    d.rcnt = at<int32_t>(pool, o.rcnt);
    d.rp_off = at<int32_t>(pool, o.rp_off);
    d.rp_src = at<int32_t>(pool, o.rp_src);
    d.rp_c = at<int64_t>(pool, o.rp_c);
    d.kx = at<int64_t>(pool, o.kx);
    d.dv = at<int64_t>(pool, o.dv);
    d.ninp = at<int32_t>(pool, o.ninp);
    d.trace = P->opt.sim_trace ? at<int64_t>(pool, o.tr) : nullptr;
    d.trace_cap = P->opt.sim_trace ? 2 * V + 2 * E + 4 : 0;
    d.trace_n = at<unsigned long long>(pool, o.trn);
    P->sim_fills.push_back({d.trace_n, 0, 8});
    P->sim_fills.push_back({d.flow8, 0, 64});
    P->sim_fills.push_back({d.resident, 0, size_t(V * n)});
    P->sim_fills.push_back({d.sent, 0, size_t(V * n)});
    P->sim_fills.push_back({d.err, 0, sizeof(DErr)});
  }
  {
    int rc = upload_fills(P->sim_fills, P->borrowed ? &thread_arena() : nullptr, 5, &P->sim_fill_dev,
                          &P->nsim_fill, msg, msglen);
    if (rc) return rc;
  }
  P->ds_dev = at<DSim>(pool, tab);
  BX_CUDA(cudaMemcpy(P->ds_dev, P->ds.data(), sizeof(DSim) * P->njobs, cudaMemcpyHostToDevice), msg, msglen);
  return BX_OK;
}

int bx_plan_simulate(bx_plan *P, int32_t mem_mode, void *stream) {
  cudaSetDevice(P->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char msg[256];
  int rc = sim_setup(P, msg, sizeof msg);
  if (rc) return rc;
  if (P->sim_mem_mode != mem_mode) {
    for (auto &d : P->ds) d.mem_mode = mem_mode;
    if (cudaMemcpy(P->ds_dev, P->ds.data(), sizeof(DSim) * P->njobs, cudaMemcpyHostToDevice) != cudaSuccess)
      return BX_RUNTIME;
    P->sim_mem_mode = mem_mode;
  }
  launch_fill(P->sim_fill_dev, P->nsim_fill, s);
  launch_simulate(P->ds_dev, P->njobs, P->dg_dev, std::max(P->maxn_all, 1), P->opt.sim_heap_cap, s);
  return launch_status();
}

int bx_plan_sim_download(bx_plan *P, void *stream, bx_sim_report *out) {
  cudaSetDevice(P->device);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (!P->sim_pool) return BX_RUNTIME;
  std::vector<DErr> errs(P->njobs);
  std::vector<int64_t> dev3n, x4(4 * static_cast<size_t>(P->njobs)), mk(P->njobs);
  std::vector<std::vector<int64_t>> d3(P->njobs);
  for (int i = 0; i < P->njobs; ++i) {
    const DSim &d = P->ds[i];
    const int V = P->hg[d.graph].V;
    d3[i].resize(3 * static_cast<size_t>(std::max(d.n, 1)));
    cudaMemcpyAsync(&errs[i], d.err, sizeof(DErr), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&x4[4 * i], d.xfer4, 32, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(&mk[i], d.makespan, 8, cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(d3[i].data(), d.dev3n, 8 * d3[i].size(), cudaMemcpyDeviceToHost, s);
    if (V > 0) cudaMemcpyAsync(out[i].start_us, d.start, 8 * size_t(V), cudaMemcpyDeviceToHost, s);
  }
  if (cudaStreamSynchronize(s) != cudaSuccess) return BX_RUNTIME;
  for (int i = 0; i < P->njobs; ++i) {
    const DSim &d = P->ds[i];
    const bx_graph &G = P->hg[d.graph];
    bx_sim_report &o = out[i];
    const DErr &e = errs[i];
    o.status = e.status;
    auto id_of = [&](int64_t meta) -> long long {
      return G.first_id ? static_cast<long long>(G.first_id[meta]) : static_cast<long long>(meta);
    };
    std::string m;
    switch (e.code) {
      case E_NONE:
        break;
      case E_SIM_MEMORY:
        m = "memory violation on device " + std::to_string(e.a) + " at t=" + std::to_string(e.b) +
            "us while holding node " + std::to_string(id_of(e.c)) + ": " + std::to_string(e.d) + " > " +
            std::to_string(P->hj[i].capacity[e.a]);
        break;
      case E_SIM_DEADLOCK:
        m = "deadlock: device " + std::to_string(e.a) + " waits forever for inputs of node " +
            std::to_string(id_of(e.c)) + "; exec_order contradicts the DAG";
        break;
      case E_SIM_STALL:
        m = "deadlock: simulation stalled";
        break;
      case E_SIM_EXEC:
        m = "exec_order disagrees with assignments";
        break;
      case E_SIM_ONCE:
        m = "placement must assign every node exactly once";
        break;
      default:
        m = "internal error code " + std::to_string(e.code);
        o.status = BX_RUNTIME;
    }
    put_msg(o.msg, sizeof o.msg, m);
    o.makespan_us = mk[i];
    o.transfer_count = x4[4 * i];
    o.transfer_bytes = x4[4 * i + 1];
    o.duplicate_transfers = x4[4 * i + 2];
    o.cache_hits = x4[4 * i + 3];
    for (int dv = 0; dv < d.n; ++dv) {
      o.peak_bytes[dv] = d3[i][3 * dv];
      o.busy_us[dv] = d3[i][3 * dv + 1];
      o.idle_us[dv] = d3[i][3 * dv + 2];
    }
  }
  return BX_OK;
}

// ---- one-shot entry points ----------------------------------------------
int bx_place(const bx_graph *graph, const bx_job *job, bx_placement *out) {
  bx_job j = *job;
  j.graph = 0;
  bx_plan *P = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = plan_create(1, graph, 1, &j, dev, nullptr, true, &P, out->msg, sizeof out->msg);
  if (rc) {
    out->status = rc;
    g_last_message = out->msg;
    return rc;
  }
  rc = bx_plan_upload(P, nullptr);
  if (!rc) rc = bx_plan_place(P, nullptr);
  if (!rc) rc = bx_plan_download(P, nullptr, out);
  g_last_message = !rc && !P->res_msg.empty() ? P->res_msg[0] : std::string(out->msg);
  if (rc) {
    out->status = rc;
    put_msg(out->msg, sizeof out->msg, std::string("CUDA error: ") + cudaGetErrorString(cudaGetLastError()));
  }
  bx_plan_destroy(P);
  return rc ? rc : out->status;
}

int bx_simulate(const bx_graph *graph, int32_t n, const int64_t *capacity, const bx_comm *cm, int32_t mem_mode,
                const int32_t *device_of, const int32_t *exec_order, const int32_t *exec_off, bx_sim_report *out) {
  return bx_simulate_ex(graph, n, capacity, cm, mem_mode, device_of, exec_order, exec_off, nullptr, out);
}

}  // extern "C"

// One-shot simulate of an external placement (bx_simulate*, bx_simulate_trace).
static int simulate_oneshot(const bx_graph *graph, int32_t n, const int64_t *capacity, const bx_comm *cm,
                            int32_t mem_mode, const int32_t *device_of, const int32_t *exec_order,
                            const int32_t *exec_off, const bx_plan_options *options, bx_sim_report *out,
                            bx_trace_event *trace, int64_t trace_cap, int64_t *trace_len) {
  if (trace_len) *trace_len = 0;
  if (n <= 0) {
    out->status = BX_VALIDATION;
    put_msg(out->msg, sizeof out->msg, "placement does not match graph or roster");
    return BX_VALIDATION;
  }
  // a job that is never placed: its placement arrays are filled from the host
  bx_job j = {};
  j.graph = 0;
  j.algo = BX_ALGO_METF;
  j.n = n;
  j.capacity = capacity;
  j.cm = *cm;
  bx_plan *P = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = plan_create(1, graph, 1, &j, dev, options, true, &P, out->msg, sizeof out->msg);
  if (rc) {
    out->status = rc;
    return rc;
  }
  const DJob &d = P->dj[0];
  const int V = graph->V;
  bool offsets_ok = exec_off[0] == 0 && exec_off[n] == V;
  for (int dv = 0; dv < n && offsets_ok; ++dv) offsets_ok = exec_off[dv] <= exec_off[dv + 1];
  if (!offsets_ok) {
    // lists that cannot hold every node exactly once never reach the device
    // buffers (sized V); the verdict is validate_placement's own
    // (simulator.cpp:78-97), decided by its first failing check
    bx_plan_destroy(P);
    out->status = BX_VALIDATION;
    const char *why = "placement must assign every node exactly once";
    for (int dv = 0; dv < n; ++dv)
      for (int x = std::max(exec_off[dv], 0); x < exec_off[dv + 1] && x < V; ++x) {
        int m = exec_order[x];
        if (m < 0 || m >= V || device_of[m] != dv) why = "exec_order disagrees with assignments";
      }
    put_msg(out->msg, sizeof out->msg, why);
    return out->status;
  }
  rc = bx_plan_upload(P, nullptr);
  if (!rc && V > 0) {
    cudaMemcpy(d.device_of, device_of, 4 * size_t(V), cudaMemcpyHostToDevice);
    cudaMemcpy(d.exec_order, exec_order, 4 * size_t(V), cudaMemcpyHostToDevice);
  }
  if (!rc) cudaMemcpy(d.exec_off, exec_off, 4 * size_t(n + 1), cudaMemcpyHostToDevice);
  if (!rc) rc = bx_plan_simulate(P, mem_mode, nullptr);
  if (!rc) rc = bx_plan_sim_download(P, nullptr, out);
  if (!rc && trace) rc = bx_plan_sim_trace(P, 0, trace, trace_cap, trace_len);
  if (rc) {
    out->status = rc;
    put_msg(out->msg, sizeof out->msg, "CUDA failure in bx_simulate");
  }
  bx_plan_destroy(P);
  return rc ? rc : out->status;
}

extern "C" {

int bx_simulate_ex(const bx_graph *graph, int32_t n, const int64_t *capacity, const bx_comm *cm, int32_t mem_mode,
                   const int32_t *device_of, const int32_t *exec_order, const int32_t *exec_off,
                   const bx_plan_options *options, bx_sim_report *out) {
  return simulate_oneshot(graph, n, capacity, cm, mem_mode, device_of, exec_order, exec_off, options, out, nullptr, 0,
                          nullptr);
}

int bx_simulate_trace(const bx_graph *graph, int32_t n, const int64_t *capacity, const bx_comm *cm, int32_t mem_mode,
                      const int32_t *device_of, const int32_t *exec_order, const int32_t *exec_off,
                      bx_sim_report *out, bx_trace_event *trace, int64_t trace_cap, int64_t *trace_len) {
  bx_plan_options o{0, -1, 0, 0, 0, -1, 1};
  return simulate_oneshot(graph, n, capacity, cm, mem_mode, device_of, exec_order, exec_off, &o, out, trace,
                          trace_cap, trace_len);
}

int bx_plan_sim_trace(bx_plan *P, int32_t job, bx_trace_event *out, int64_t cap, int64_t *len) {
  cudaSetDevice(P->device);
  *len = 0;
  if (!P->sim_pool || job < 0 || job >= P->njobs || !P->ds[job].trace) return BX_VALIDATION;
  const DSim &d = P->ds[job];
  unsigned long long cnt = 0;
  if (cudaMemcpy(&cnt, d.trace_n, 8, cudaMemcpyDeviceToHost) != cudaSuccess) return BX_RUNTIME;
  const int64_t have = std::min<int64_t>(static_cast<int64_t>(cnt), d.trace_cap);
  const int64_t m = std::min<int64_t>(have, cap);
  std::vector<int64_t> raw(4 * static_cast<size_t>(m));
  if (m > 0 && cudaMemcpy(raw.data(), d.trace, 32 * size_t(m), cudaMemcpyDeviceToHost) != cudaSuccess)
    return BX_RUNTIME;
  const bx_graph &G = P->hg[d.graph];
  for (int64_t i = 0; i < m; ++i) {
    const int64_t meta = raw[4 * i + 3];
    out[i].time_us = raw[4 * i];
    out[i].device = static_cast<int32_t>(raw[4 * i + 1]);
    out[i].event = static_cast<int32_t>(raw[4 * i + 2]);
    out[i].node = G.first_id ? G.first_id[meta] : meta;  // base_id(meta), simulator.cpp:56-58
  }
  *len = have;
  return have > cap ? BX_VALIDATION : BX_OK;
}

int bx_round_extract(int32_t V, int32_t E, const int32_t *esrc, const int32_t *edst, const double *x,
                     double threshold, int32_t *fav_child, int32_t *fav_parent, int32_t *stats2, char *msg,
                     int msglen) {
  if (threshold <= 0 || threshold >= 0.5) {  // lp.cpp:282-284
    put_msg(msg, msglen, "rounding threshold must lie in (0, 0.5)");
    return BX_VALIDATION;
  }
  if (bx_device_count() <= 0) {
    put_msg(msg, msglen, "no CUDA device: the B200 placement engine has no CPU fallback");
    return BX_RUNTIME;
  }
  for (int e = 0; e < E; ++e)
    if (esrc[e] < 0 || esrc[e] >= V || edst[e] < 0 || edst[e] >= V) {
      put_msg(msg, msglen, "edge endpoint outside the graph");
      return BX_VALIDATION;
    }
  Layout L;
  size_t o_src = L.take<int32_t>(E), o_dst = L.take<int32_t>(E), o_x = L.take<double>(E);
  size_t o_smin = L.take<unsigned long long>(V), o_dmin = L.take<unsigned long long>(V);
  size_t o_speer = L.take<int32_t>(V), o_dpeer = L.take<int32_t>(V);
  size_t o_cs = L.take<int32_t>(V), o_cd = L.take<int32_t>(V), o_best = L.take<int32_t>(V);
  size_t o_fc = L.take<int32_t>(V), o_fp = L.take<int32_t>(V), o_st = L.take<int32_t>(2);
  void *pool = nullptr;
  BX_CUDA(cudaMalloc(&pool, L.off), msg, msglen);
  XCtx c;
  c.V = V;
  c.E = E;
  c.esrc = at<int32_t>(pool, o_src);
  c.edst = at<int32_t>(pool, o_dst);
  c.x = at<double>(pool, o_x);
  c.thr = threshold;
  c.src_min = at<unsigned long long>(pool, o_smin);
  c.dst_min = at<unsigned long long>(pool, o_dmin);
  c.src_peer = at<int32_t>(pool, o_speer);
  c.dst_peer = at<int32_t>(pool, o_dpeer);
  c.cnt_src = at<int32_t>(pool, o_cs);
  c.cnt_dst = at<int32_t>(pool, o_cd);
  c.best_edge = at<int32_t>(pool, o_best);
  c.fav_child = at<int32_t>(pool, o_fc);
  c.fav_parent = at<int32_t>(pool, o_fp);
  c.stats2 = at<int32_t>(pool, o_st);
  cudaError_t ce = cudaSuccess;
  auto chk = [&](cudaError_t e) {
    if (ce == cudaSuccess) ce = e;
  };
  if (E > 0) {
    chk(cudaMemcpy(const_cast<int32_t *>(c.esrc), esrc, 4 * size_t(E), cudaMemcpyHostToDevice));
    chk(cudaMemcpy(const_cast<int32_t *>(c.edst), edst, 4 * size_t(E), cudaMemcpyHostToDevice));
    chk(cudaMemcpy(const_cast<double *>(c.x), x, 8 * size_t(E), cudaMemcpyHostToDevice));
  }
  chk(cudaMemset(c.src_min, 0xff, 8 * size_t(V)));
  chk(cudaMemset(c.dst_min, 0xff, 8 * size_t(V)));
  chk(cudaMemset(c.src_peer, 0x7f, 4 * size_t(V)));
  chk(cudaMemset(c.dst_peer, 0x7f, 4 * size_t(V)));
  chk(cudaMemset(c.cnt_src, 0, 4 * size_t(V)));
  chk(cudaMemset(c.cnt_dst, 0, 4 * size_t(V)));
  chk(cudaMemset(c.best_edge, 0xff, 4 * size_t(V)));
  chk(cudaMemset(c.fav_child, 0xff, 4 * size_t(V)));
  chk(cudaMemset(c.fav_parent, 0xff, 4 * size_t(V)));
  chk(cudaMemset(c.stats2, 0, 8));
  if (ce == cudaSuccess && V > 0) {
    launch_extract(c, nullptr);
    chk(cudaGetLastError());
  }
  if (V > 0) {
    chk(cudaMemcpy(fav_child, c.fav_child, 4 * size_t(V), cudaMemcpyDeviceToHost));
    chk(cudaMemcpy(fav_parent, c.fav_parent, 4 * size_t(V), cudaMemcpyDeviceToHost));
  }
  chk(cudaMemcpy(stats2, c.stats2, 8, cudaMemcpyDeviceToHost));
  cudaFree(pool);
  if (ce != cudaSuccess) {
    put_msg(msg, msglen, std::string("CUDA error: ") + cudaGetErrorString(ce));
    return BX_RUNTIME;
  }
  put_msg(msg, msglen, "");
  return BX_OK;
}

}  // extern "C"

// ---- exhaustive oracle (oracle.hpp:29-34, oracle.cpp:17-212) ---------------------
// The exact minimum makespan over every canonical device assignment and every
// DAG-consistent global order (restricted per device), each pair scored by
// the GPU simulator (K4 / K4f) in batches of one plan: the placements are
// written into the plan's output region, simulated, and a reduction kernel
// keeps the batch minimum. Pruning as the reference (static memory, the
// assignment's load floor, the global lower bound) only skips pairs that
// cannot change the minimum.
namespace bx {
__global__ void k_oracle_min(const DSim *sims, int count, unsigned long long *best, unsigned int *bad) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x) {
    const DSim &d = sims[i];
    const int st = d.err->status;
    if (st == kOk) atomicMin(best, static_cast<unsigned long long>(*d.makespan));
    else if (!(st == kInfeasible && d.err->code == E_SIM_MEMORY)) atomicAdd(bad, 1u);  // memory: skipped
  }
}

// Fast path (parallel comm, no capacity, every node k > 0): a node's start is
// max(its device predecessor's finish, max over remote parents of finish +
// c(parent, device)), c = comm_time of the largest tensor the parent sends to
// that device (K4f's recurrence, simulator.cpp:156-181), so walking a
// DAG-consistent global order gives the simulator's schedule for the
// per-device orders it induces. One warp per canonical assignment (its
// transfer-time table built once), lanes over the global orders, a
// warp-minimum then one atomicMin per warp. Every (assignment, order) pair
// is scored, so no pruning is needed.
constexpr int kOrMaxV = 16, kOrMaxN = 8;
__device__ __forceinline__ int64_t omax(int64_t a, int64_t b) { return a > b ? a : b; }
__global__ void k_oracle_fast(int V, int n, int64_t A, int64_t X, const uint8_t *asg, const uint8_t *ext,
                              const int32_t *in_off, const int32_t *in_src, const int32_t *out_off,
                              const int32_t *edst, const int64_t *bytes, const int64_t *k, double ic, double pb,
                              unsigned long long *best) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5;
  for (int64_t a = warp; a < A; a += nwarps) {
    int dev[kOrMaxV];
    int64_t ct[kOrMaxV][kOrMaxN];
    for (int i = 0; i < V; ++i) dev[i] = asg[a * V + i];
    for (int i = 0; i < V; ++i) {
      int64_t mb[kOrMaxN];
      for (int d = 0; d < n; ++d) mb[d] = 0;  // the reference's per-destination slot starts at 0
      for (int e = out_off[i]; e < out_off[i + 1]; ++e) {
        const int dc = dev[edst[e]];
        if (dc != dev[i]) mb[dc] = omax(mb[dc], bytes[e]);
      }
      for (int d = 0; d < n; ++d) ct[i][d] = comm_time_exact(ic, pb, mb[d]);
    }
    unsigned long long mine = ~0ull;
    for (int64_t x = lane; x < X; x += 32) {
      int64_t fin[kOrMaxV], dfree[kOrMaxN];
      for (int d = 0; d < n; ++d) dfree[d] = 0;
      int64_t mk = 0;
      for (int r = 0; r < V; ++r) {
        const int j = ext[x * V + r], dj = dev[j];
        int64_t t = dfree[dj];
        for (int y = in_off[j]; y < in_off[j + 1]; ++y) {
          const int i = in_src[y];
          t = omax(t, dev[i] == dj ? fin[i] : fin[i] + ct[i][dj]);
        }
        fin[j] = t + k[j];
        dfree[dj] = fin[j];
        mk = omax(mk, fin[j]);
      }
      mine = min(mine, static_cast<unsigned long long>(mk));
    }
    const unsigned hi = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(mine >> 32));
    const unsigned lo = __reduce_min_sync(0xffffffffu, static_cast<unsigned>(mine >> 32) == hi
                                                           ? static_cast<unsigned>(mine) : 0xffffffffu);
    if (lane == 0) atomicMin(best, (static_cast<unsigned long long>(hi) << 32) | lo);
  }
}
}  // namespace bx

extern "C" int bx_oracle_makespan(const bx_graph *graph, int32_t n, const bx_comm *cm, int64_t capacity,
                                  int32_t mem_mode, int32_t max_nodes, int32_t max_devices, int64_t max_extensions,
                                  int64_t *out_us, char *msg, int msglen) {
  *out_us = 0;
  const int V = graph->V;
  if (V > max_nodes) {
    put_msg(msg, msglen, "instance too large: " + std::to_string(V) + " nodes > " + std::to_string(max_nodes));
    return BX_INFEASIBLE;
  }
  if (n < 1 || n > max_devices) {
    put_msg(msg, msglen, "instance too large: " + std::to_string(n) + " devices > " + std::to_string(max_devices));
    return BX_INFEASIBLE;
  }
  const bool limited = capacity >= 0;
  const int64_t cap = limited ? capacity : INT64_MAX / 4;
  // every DAG-consistent global order (enumerate_extensions, oracle.cpp:23-54)
  std::vector<std::vector<int>> ext;
  {
    std::vector<int> pending(V, 0), prefix;
    for (int e = 0; e < graph->E; ++e) pending[graph->edst[e]]++;
    bool too_many = false;
    std::function<void()> rec = [&]() {
      if (too_many) return;
      if (static_cast<int>(prefix.size()) == V) {
        if (static_cast<int64_t>(ext.size()) >= max_extensions) {
          too_many = true;
          return;
        }
        ext.push_back(prefix);
        return;
      }
      for (int j = 0; j < V && !too_many; ++j) {
        if (pending[j] != 0) continue;
        pending[j] = -1;
        for (int e = graph->out_off[j]; e < graph->out_off[j + 1]; ++e) pending[graph->edst[e]]--;
        prefix.push_back(j);
        rec();
        prefix.pop_back();
        for (int e = graph->out_off[j]; e < graph->out_off[j + 1]; ++e) pending[graph->edst[e]]++;
        pending[j] = 0;
      }
    };
    rec();
    if (too_many) {
      put_msg(msg, msglen,
              "instance too large: more than " + std::to_string(max_extensions) + " execution orders to enumerate");
      return BX_INFEASIBLE;
    }
  }
  // canonical assignments: labels in first-use order (oracle.cpp:58-73)
  std::vector<std::vector<int>> asg;
  {
    std::vector<int> a(V, 0);
    std::function<void(int, int)> rec = [&](int i, int used) {
      if (i == V) {
        asg.push_back(a);
        return;
      }
      const int limit = std::min(n, used + 1);
      for (int d = 0; d < limit; ++d) {
        a[i] = d;
        rec(i + 1, std::max(used, d + 1));
      }
    };
    rec(0, 0);
  }
  // lower bound: critical path and the work bound (oracle.cpp:103-105)
  int64_t cp = 0;
  {
    const int rc = bx_critical_path_us(graph, &cp, msg, msglen);
    if (rc) return rc;
  }
  int64_t total = 0;
  for (int j = 0; j < V; ++j) total += graph->compute_us[j];
  const int64_t lower = std::max(cp, (total + n - 1) / n);
  constexpr uint64_t kNone = ~0ull;
  uint64_t best = kNone;
  if (ext.empty()) {  // V == 0: one (empty) schedule
    put_msg(msg, msglen, "");
    *out_us = 0;
    return BX_OK;
  }
  // fast path: parallel comm, no capacity, every node k > 0, small enough
  {
    bool ok = cm->mode == BX_COMM_PARALLEL && !limited && V <= bx::kOrMaxV && n <= bx::kOrMaxN;
    for (int v = 0; v < V && ok; ++v) ok = graph->compute_us[v] > 0;
    for (int e = 0; e < graph->E && ok; ++e) ok = graph->tensor_bytes[e] >= 0;
    if (ok) {
      const int64_t A = static_cast<int64_t>(asg.size()), X = static_cast<int64_t>(ext.size());
      std::vector<uint8_t> ha(A * V), hx(X * V);
      for (int64_t a = 0; a < A; ++a)
        for (int v = 0; v < V; ++v) ha[a * V + v] = static_cast<uint8_t>(asg[a][v]);
      for (int64_t x = 0; x < X; ++x)
        for (int v = 0; v < V; ++v) hx[x * V + v] = static_cast<uint8_t>(ext[x][v]);
      std::vector<int32_t> in_src(std::max(graph->E, 1));
      for (int x = 0; x < graph->E; ++x) in_src[x] = graph->esrc[graph->in_edge[x]];
      char *d = nullptr;
      const size_t bA = ha.size(), bX = hx.size(), bV1 = 4 * size_t(V + 1), bE = std::max(graph->E, 1);
      const size_t total = 256 + bA + bX + 2 * bV1 + 4 * bE * 2 + 8 * bE + 8 * size_t(V) + 64 * 8;
      if (cudaMalloc(&d, total) != cudaSuccess) {
        put_msg(msg, msglen, "CUDA failure in the oracle");
        return BX_RUNTIME;
      }
      size_t o = 0;
      auto take = [&](size_t b) {
        char *p = d + o;
        o += (b + 15) & ~size_t(15);
        return p;
      };
      unsigned long long *dbest = reinterpret_cast<unsigned long long *>(take(8));
      uint8_t *da = reinterpret_cast<uint8_t *>(take(bA)), *dx = reinterpret_cast<uint8_t *>(take(bX));
      int32_t *dio = reinterpret_cast<int32_t *>(take(bV1)), *doo = reinterpret_cast<int32_t *>(take(bV1));
      int32_t *dis = reinterpret_cast<int32_t *>(take(4 * bE)), *ded = reinterpret_cast<int32_t *>(take(4 * bE));
      int64_t *dby = reinterpret_cast<int64_t *>(take(8 * bE)), *dk = reinterpret_cast<int64_t *>(take(8 * size_t(V)));
      const unsigned long long init = ~0ull;
      bool good = cudaMemcpy(dbest, &init, 8, cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(da, ha.data(), bA, cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(dx, hx.data(), bX, cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(dio, graph->in_off, bV1, cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(doo, graph->out_off, bV1, cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(dis, in_src.data(), 4 * size_t(graph->E), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(ded, graph->edst, 4 * size_t(graph->E), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(dby, graph->tensor_bytes, 8 * size_t(graph->E), cudaMemcpyHostToDevice) == cudaSuccess &&
                  cudaMemcpy(dk, graph->compute_us, 8 * size_t(V), cudaMemcpyHostToDevice) == cudaSuccess;
      unsigned long long res = ~0ull;
      if (good) {
        const int64_t warps = std::min<int64_t>(A, 148 * 64);
        bx::k_oracle_fast<<<static_cast<int>((warps * 32 + 255) / 256), 256>>>(
            V, n, A, X, da, dx, dio, dis, doo, ded, dby, dk, cm->intercept_us, cm->us_per_byte, dbest);
        good = cudaMemcpy(&res, dbest, 8, cudaMemcpyDeviceToHost) == cudaSuccess;
      }
      cudaFree(d);
      if (!good) {
        put_msg(msg, msglen, "CUDA failure in the oracle");
        return BX_RUNTIME;
      }
      *out_us = static_cast<int64_t>(res);
      put_msg(msg, msglen, "");
      return BX_OK;
    }
  }
  // one plan, B identical jobs; placements go into its output region
  const int64_t pairs_total = static_cast<int64_t>(asg.size()) * static_cast<int64_t>(ext.size());
  const int B = static_cast<int>(std::min<int64_t>(pairs_total, 8192));
  std::vector<int64_t> caps(n, cap);
  bx_job j = {};
  j.graph = 0;
  j.algo = BX_ALGO_METF;
  j.n = n;
  j.capacity = caps.data();
  j.cm = *cm;
  std::vector<bx_job> jobs(B, j);
  bx_plan *P = nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = plan_create(1, graph, B, jobs.data(), dev, nullptr, false, &P, msg, msglen);
  if (rc) return rc;
  if (bx_plan_upload(P, nullptr) != BX_OK) {  // the graph and the capacities
    bx_plan_destroy(P);
    put_msg(msg, msglen, "CUDA failure in the oracle");
    return BX_RUNTIME;
  }
  unsigned long long *dbest = nullptr;
  unsigned int *dbad = nullptr;
  char *dscratch = nullptr;
  if (cudaMalloc(&dscratch, 16) != cudaSuccess) {
    bx_plan_destroy(P);
    put_msg(msg, msglen, "CUDA failure in the oracle");
    return BX_RUNTIME;
  }
  dbest = reinterpret_cast<unsigned long long *>(dscratch);
  dbad = reinterpret_cast<unsigned int *>(dscratch + 8);
  char *H = static_cast<char *>(P->host_out);
  int filled = 0;
  bool failed = false, done = false;
  auto run_batch = [&]() {
    if (filled == 0 || failed) return;
    for (int i = filled; i < B; ++i) {  // unused slots repeat the first pair of the batch
      std::memcpy(H + P->out_off[i].dev, H + P->out_off[0].dev, 4 * size_t(V));
      std::memcpy(H + P->out_off[i].eo, H + P->out_off[0].eo, 4 * size_t(V));
      std::memcpy(H + P->out_off[i].eoff, H + P->out_off[0].eoff, 4 * size_t(n + 1));
    }
    unsigned long long init[2] = {kNone, 0};
    if (cudaMemcpy(P->dev_out, H, P->out_bytes, cudaMemcpyHostToDevice) != cudaSuccess ||
        cudaMemcpy(dscratch, init, 16, cudaMemcpyHostToDevice) != cudaSuccess ||
        bx_plan_simulate(P, mem_mode, nullptr) != BX_OK) {
      failed = true;
      return;
    }
    bx::k_oracle_min<<<(B + 255) / 256, 256>>>(P->ds_dev, B, dbest, dbad);
    unsigned long long res[2];
    if (cudaMemcpy(res, dscratch, 16, cudaMemcpyDeviceToHost) != cudaSuccess || (res[1] & 0xffffffffull)) {
      failed = true;
      return;
    }
    best = std::min<uint64_t>(best, res[0]);
    filled = 0;
    if (best != kNone && static_cast<int64_t>(best) <= lower) done = true;
  };
  std::vector<int64_t> need(n), load(n);
  for (size_t a = 0; a < asg.size() && !done && !failed; ++a) {
    const std::vector<int> &as = asg[a];
    if (limited) {  // static memory (perm) before anything runs (oracle.cpp:118-128)
      std::fill(need.begin(), need.end(), 0);
      for (int v = 0; v < V; ++v) need[as[v]] += graph->perm_bytes[v];
      bool over = false;
      for (int d = 0; d < n; ++d) over |= need[d] > cap;
      if (over) continue;
    }
    std::fill(load.begin(), load.end(), 0);
    for (int v = 0; v < V; ++v) load[as[v]] += graph->compute_us[v];
    const int64_t floor_a = std::max(lower, *std::max_element(load.begin(), load.end()));
    if (best != kNone && floor_a >= static_cast<int64_t>(best)) continue;  // cannot beat the incumbent
    for (size_t x = 0; x < ext.size() && !done && !failed; ++x) {
      const bx_plan::OOff &o = P->out_off[filled];
      int32_t *dv = reinterpret_cast<int32_t *>(H + o.dev), *eo = reinterpret_cast<int32_t *>(H + o.eo),
              *eoff = reinterpret_cast<int32_t *>(H + o.eoff);
      std::fill(eoff, eoff + n + 1, 0);
      for (int v = 0; v < V; ++v) {
        dv[v] = as[v];
        eoff[as[v] + 1]++;
      }
      for (int d = 0; d < n; ++d) eoff[d + 1] += eoff[d];
      std::vector<int> at(eoff, eoff + n);
      for (int v : ext[x]) eo[at[as[v]]++] = v;
      if (++filled == B) run_batch();
    }
  }
  run_batch();
  cudaFree(dscratch);
  bx_plan_destroy(P);
  if (failed) {
    put_msg(msg, msglen, "CUDA failure or unexpected simulator error in the oracle");
    return BX_RUNTIME;
  }
  if (best == kNone) {
    put_msg(msg, msglen, "no device assignment fits the memory capacities");
    return BX_INFEASIBLE;
  }
  *out_us = static_cast<int64_t>(best);
  put_msg(msg, msglen, "");
  return BX_OK;
}

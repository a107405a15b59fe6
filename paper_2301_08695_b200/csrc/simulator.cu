// K4 — the event-driven makespan simulator (simulate, proj/src/simulator.cpp
// :26-278) and K3 — favourite-child extraction (round_and_extract,
// proj/src/lp.cpp:280-326), for sm_100a.
//
// K4: one warp per (graph, placement) problem. Events are processed in the
// reference's heap order (t, kind{finish 0 < xfer_done 1 < start 2}, a, b)
// (simulator.cpp:14-24); the heap stores (t, packed(kind, a, b)) pairs so one
// 128-bit compare orders them. Lane 0 owns the heap; the whole warp scans the
// out-edge lists (input-residency counters, the per-destination max bytes,
// GraphStatic releases). K4f (further down) replaces the event loop for
// parallel comm mode without zero-duration nodes.
#include <algorithm>
#include <cstdlib>

#include "bx_device.cuh"

namespace bx {

constexpr unsigned kFullS = 0xffffffffu;

__device__ __forceinline__ int64_t smax(int64_t a, int64_t b) { return a > b ? a : b; }

// packed = kind << 58 | a << 20 | b   (a < 2^38, b < 2^20)
__device__ __forceinline__ int64_t pack_ev(int kind, int a, int b) {
  return (static_cast<int64_t>(kind) << 58) | (static_cast<int64_t>(a) << 20) | static_cast<int64_t>(b);
}

// The event heap starts in the warp's shared-memory slice (the live event
// set is small: running nodes, transfers in flight, queued starts) and moves
// to its global-memory arrays the first time it outgrows the slice.
struct Heap {
  int64_t *t, *k;
  int64_t size, cap;
  int64_t *gt, *gk;  // global arrays (capacity 2n + E + 16, never outgrown)
  bool spilled;
  __device__ bool less(int64_t x, int64_t y) const { return t[x] < t[y] || (t[x] == t[y] && k[x] < k[y]); }
  __device__ void swap(int64_t x, int64_t y) {
    int64_t a = t[x], b = k[x];
    t[x] = t[y];
    k[x] = k[y];
    t[y] = a;
    k[y] = b;
  }
  __device__ void push(int64_t tt, int64_t kk) {
    if (size == cap && !spilled) {
      for (int64_t x = 0; x < size; ++x) {
        gt[x] = t[x];
        gk[x] = k[x];
      }
      t = gt;
      k = gk;
      spilled = true;
    }
    int64_t i = size++;
    t[i] = tt;
    k[i] = kk;
    while (i > 0) {
      int64_t p = (i - 1) >> 1;
      if (!less(i, p)) break;
      swap(i, p);
      i = p;
    }
  }
  __device__ void pop(int64_t &tt, int64_t &kk) {
    tt = t[0];
    kk = k[0];
    --size;
    t[0] = t[size];
    k[0] = k[size];
    int64_t i = 0;
    while (true) {
      int64_t l = 2 * i + 1, r = l + 1, m = i;
      if (l < size && less(l, m)) m = l;
      if (r < size && less(r, m)) m = r;
      if (m == i) break;
      swap(i, m);
      i = m;
    }
  }
};

struct SimCtx {
  DSim s;
  DGraph g;
  int V, n;
  Heap h;
  int lane;
};

// inputs_resident (simulator.cpp:100-111) as a counter: ninp[j] starts at
// j's in-edge count and drops when a same-device parent finishes or a
// parent's tensor lands on j's device (each (parent, device) transfer is sent
// exactly once), so the test at try_start is one load instead of a scan.
__device__ __forceinline__ void inputs_landed(const SimCtx &c, int i, int dev) {
  for (int y = c.g.out_off[i] + c.lane; y < c.g.out_off[i + 1]; y += 32) {
    const int ch = c.g.edst[y];
    if (c.s.device_of[ch] == dev) atomicSub(&c.s.ninp[ch], 1);
  }
  __syncwarp();
}

// try_start (simulator.cpp:113-119). Warp-uniform control flow; lane 0 pushes.
__device__ void try_start(SimCtx &c, int dev, int64_t now) {
  if (c.s.busy[dev]) return;
  int len = c.s.exec_off[dev + 1] - c.s.exec_off[dev];
  int q = c.s.qpos[dev];
  if (q >= len) return;
  int j = c.s.exec_order[c.s.exec_off[dev] + q];
  if (c.s.start_q[j]) return;
  if (c.s.ninp[j] != 0) return;
  __syncwarp();
  if (c.lane == 0) {
    c.s.start_q[j] = 1;
    c.h.push(now, pack_ev(2, j, 0));
  }
  c.h.size = __shfl_sync(kFullS, c.h.size, 0);
  __syncwarp();
}

// Sim::trace (simulator.cpp:60-64): one record per event in processing
// order; event 0 start, 1 finish, 2 xfer_begin, 3 xfer_end. Lane 0 only.
__device__ __forceinline__ void trace_ev(const DSim &s, int64_t t, int dev, int ev, int meta) {
  if (!s.trace) return;
  const unsigned long long i = *s.trace_n;
  if (static_cast<int64_t>(i) < s.trace_cap) {
    int64_t *r = s.trace + 4 * i;
    r[0] = t;
    r[1] = dev;
    r[2] = ev;
    r[3] = meta;
  }
  *s.trace_n = i + 1;
}

// charge (simulator.cpp:66-76); returns false on a violation (error set).
__device__ bool charge(SimCtx &c, int dev, int64_t delta, int64_t t, int meta) {
  int64_t m = c.s.mem[dev] + delta;
  c.s.mem[dev] = m;
  if (m > c.s.peak[dev]) c.s.peak[dev] = m;
  if (m > c.s.cap[dev]) {
    DErr *e = c.s.err;
    e->status = kInfeasible;
    e->code = E_SIM_MEMORY;
    e->a = dev;
    e->b = t;
    e->c = meta;
    e->d = m;
    return false;
  }
  return true;
}

template <int kWarps>
__global__ void __launch_bounds__(32 * kWarps) k_simulate(const DSim *sims, int nsims, const DGraph *graphs,
                                                         int sim_heap_cap, int dev_slots) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sid = blockIdx.x * kWarps + warp;
  if (sid >= nsims) return;
  SimCtx c;
  c.s = sims[sid];
  c.g = graphs[c.s.graph];
  c.V = c.g.V;
  c.n = c.s.n;
  c.lane = lane;
  // without zero-duration nodes or a trace, parallel comm mode belongs to K4f
  // and sequential comm mode on <= 32 devices to its sequencer (the first prep
  // pass flags those)
  if ((c.s.mode == 1 || (c.s.mode == 0 && c.n <= 32)) && !c.s.flow8[0]) return;
  {
    extern __shared__ int64_t sim_heap_smem[];
    const int64_t scap = static_cast<int64_t>(sim_heap_cap);
    // per-device state in this warp's shared-memory slice (after all heaps)
    // when the roster fits: every event reads and writes it on lane 0's chain
    if (dev_slots >= c.n && dev_slots > 0) {
      int64_t *base = sim_heap_smem + static_cast<int64_t>(kWarps) * 2 * scap +
                      static_cast<int64_t>(warp) * 6 * dev_slots;
      c.s.mem = base;
      c.s.peak = base + dev_slots;
      c.s.xfree = base + 2 * dev_slots;
      c.s.dest_bytes = base + 3 * dev_slots;
      c.s.qpos = reinterpret_cast<int32_t *>(base + 4 * dev_slots);
      c.s.dest_cnt = c.s.qpos + dev_slots;
      c.s.busy = reinterpret_cast<uint8_t *>(base + 5 * dev_slots);
    }
    c.h.gt = c.s.heap_t;
    c.h.gk = c.s.heap_k;
    c.h.size = 0;
    if (scap > 0) {
      c.h.t = sim_heap_smem + static_cast<int64_t>(warp) * 2 * scap;
      c.h.k = c.h.t + scap;
      c.h.cap = scap;
      c.h.spilled = false;
    } else {
      c.h.t = c.h.gt;
      c.h.k = c.h.gk;
      c.h.cap = INT64_MAX;
      c.h.spilled = true;
    }
  }
  const int V = c.V, n = c.n;
  DErr *err = c.s.err;

  // ---- validate_placement (simulator.cpp:78-97) ---------------------------
  bool bad_exec = false;
  for (int j = lane; j < V; j += 32) c.s.seen[j] = 0;
  __syncwarp();
  for (int d = 0; d < n; ++d) {
    for (int x = c.s.exec_off[d] + lane; x < c.s.exec_off[d + 1]; x += 32) {
      int m = c.s.exec_order[x];
      if (m < 0 || m >= V || c.s.device_of[m] != d) bad_exec = true;
      else atomicAdd(&c.s.seen[m], 1);
    }
  }
  if (__any_sync(kFullS, bad_exec)) {
    if (lane == 0) {
      err->status = kValidation;
      err->code = E_SIM_EXEC;
    }
    return;
  }
  __syncwarp();
  bool bad_once = false;
  for (int j = lane; j < V; j += 32) {
    int d = c.s.device_of[j];
    if (d < 0 || d >= n || c.s.seen[j] != 1) bad_once = true;
  }
  if (__any_sync(kFullS, bad_once)) {
    if (lane == 0) {
      err->status = kValidation;
      err->code = E_SIM_ONCE;
    }
    return;
  }

  // ---- state --------------------------------------------------------------
  for (int d = lane; d < n; d += 32) {
    c.s.mem[d] = 0;
    c.s.peak[d] = 0;
    c.s.xfree[d] = 0;
    c.s.qpos[d] = 0;
    c.s.busy[d] = 0;
    c.s.dest_bytes[d] = 0;
    c.s.dest_cnt[d] = 0;
  }
  for (int j = lane; j < V; j += 32) {
    c.s.consumers_left[j] = c.g.out_off[j + 1] - c.g.out_off[j];
    c.s.ninp[j] = c.g.in_off[j + 1] - c.g.in_off[j];
    c.s.finished[j] = 0;
    c.s.start_q[j] = 0;
    c.s.start[j] = 0;
  }
  __syncwarp();
  // permanent memory up front, device by device in exec order (:209-214)
  int ok = 1;
  if (lane == 0) {
    for (int d = 0; d < n && ok; ++d)
      for (int x = c.s.exec_off[d]; x < c.s.exec_off[d + 1] && ok; ++x) {
        int m = c.s.exec_order[x];
        ok = charge(c, d, c.g.perm[m], 0, m);
      }
  }
  ok = __shfl_sync(kFullS, ok, 0);
  if (!ok) return;
  __syncwarp();
  for (int d = 0; d < n; ++d) try_start(c, d, 0);

  int64_t makespan = 0, xcount = 0, xbytes = 0, dups = 0, hits = 0;
  int finished_count = 0;
  while (c.h.size > 0) {
    int64_t t = 0, pk = 0;
    if (lane == 0) c.h.pop(t, pk);
    t = __shfl_sync(kFullS, t, 0);
    pk = __shfl_sync(kFullS, pk, 0);
    c.h.size = __shfl_sync(kFullS, c.h.size, 0);
    const int kind = static_cast<int>(pk >> 58);
    const int a = static_cast<int>((pk >> 20) & ((int64_t(1) << 38) - 1));
    const int b = static_cast<int>(pk & ((1 << 20) - 1));
    __syncwarp();
    if (kind == 2) {
      // run_start (:121-131)
      int dev = c.s.device_of[a];
      if (lane == 0) {
        c.s.busy[dev] = 1;
        c.s.start[a] = t;
        ok = charge(c, dev, c.g.temp[a] + c.g.outb[a], t, a);
        if (ok) trace_ev(c.s, t, dev, 0, a);
        if (ok) c.h.push(t + c.g.k[a], pack_ev(0, a, 0));
      }
      ok = __shfl_sync(kFullS, ok, 0);
      if (!ok) return;
      c.h.size = __shfl_sync(kFullS, c.h.size, 0);
      __syncwarp();
    } else if (kind == 0) {
      // run_finish (:133-184)
      const int j = a;
      const int dev = c.s.device_of[j];
      ++finished_count;
      makespan = smax(makespan, t);
      if (lane == 0) {
        trace_ev(c.s, t, dev, 1, j);
        c.s.busy[dev] = 0;
        c.s.qpos[dev]++;
        c.s.finished[j] = 1;
        c.s.mem[dev] -= c.g.temp[j];
        if (c.s.mem_mode == 0 && c.s.consumers_left[j] == 0) c.s.mem[dev] -= c.g.outb[j];
      }
      __syncwarp();
      if (c.s.mem_mode == 0) {
        // parents whose last consumer this was free their outputs; only
        // decrements, checked at starts, so the lanes may take them in any order
        for (int x = c.g.in_off[j] + lane; x < c.g.in_off[j + 1]; x += 32) {
          const int i = c.g.esrc[c.g.in_edge[x]];
          if (atomicSub(&c.s.consumers_left[i], 1) == 1)
            atomicAdd(reinterpret_cast<unsigned long long *>(&c.s.mem[c.s.device_of[i]]),
                      static_cast<unsigned long long>(-c.g.outb[i]));
        }
        __syncwarp();
      }
      // destinations: max bytes per remote consumer device
      int remote = 0;
      for (int y = c.g.out_off[j] + lane; y < c.g.out_off[j + 1]; y += 32) {
        int cdev = c.s.device_of[c.g.edst[y]];
        if (cdev == dev) continue;
        ++remote;
        c.s.dest_cnt[cdev] = 1;
        // the reference's per-destination slot starts at 0 (std::map value)
        atomicMax(reinterpret_cast<unsigned long long *>(&c.s.dest_bytes[cdev]),
                  static_cast<unsigned long long>(c.g.ebytes[y] > 0 ? c.g.ebytes[y] : 0));
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) remote += __shfl_xor_sync(kFullS, remote, o);
      __syncwarp();
      int distinct = 0;
      if (remote > 0 && lane == 0) {
        for (int cdev = 0; cdev < n; ++cdev) {
          if (!c.s.dest_cnt[cdev]) continue;
          int64_t bytes = c.s.dest_bytes[cdev];
          c.s.dest_bytes[cdev] = 0;
          c.s.dest_cnt[cdev] = 0;
          ++distinct;
          int64_t key = static_cast<int64_t>(j) * n + cdev;
          if (c.s.resident[key] || c.s.sent[key]) {
            ++dups;
            continue;
          }
          c.s.sent[key] = 1;
          int64_t cc = comm_time_exact(c.s.ic, c.s.pb, bytes);
          int64_t begin = t;
          if (c.s.mode == 0) {
            begin = smax(t, smax(c.s.xfree[dev], c.s.xfree[cdev]));
            c.s.xfree[dev] = begin + cc;
            c.s.xfree[cdev] = begin + cc;
          }
          ++xcount;
          xbytes += bytes;
          trace_ev(c.s, begin, dev, 2, j);
          c.h.push(begin + cc, pack_ev(1, j, cdev));
        }
      }
      distinct = __shfl_sync(kFullS, distinct, 0);
      hits += remote - distinct;
      c.h.size = __shfl_sync(kFullS, c.h.size, 0);
      __syncwarp();
      inputs_landed(c, j, dev);  // same-device consumers now hold j's output
      try_start(c, dev, t);
    } else {
      // run_xfer_done (:186-190)
      if (lane == 0) {
        c.s.resident[static_cast<int64_t>(a) * n + b] = 1;
        trace_ev(c.s, t, b, 3, a);
      }
      __syncwarp();
      inputs_landed(c, a, b);
      try_start(c, b, t);
    }
  }
  if (finished_count != V) {
    // deadlock (:234-246): first device with work left names its head node
    if (lane == 0) {
      err->status = kValidation;
      err->code = E_SIM_STALL;
      for (int d = 0; d < n; ++d) {
        int len = c.s.exec_off[d + 1] - c.s.exec_off[d];
        if (c.s.qpos[d] < len) {
          err->code = E_SIM_DEADLOCK;
          err->a = d;
          err->c = c.s.exec_order[c.s.exec_off[d] + c.s.qpos[d]];
          break;
        }
      }
    }
    return;
  }
  // per-device busy / idle (:248-255)
  for (int d = 0; d < n; ++d) {
    int64_t busy = 0;
    for (int x = c.s.exec_off[d] + lane; x < c.s.exec_off[d + 1]; x += 32) busy += c.g.k[c.s.exec_order[x]];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) busy += __shfl_xor_sync(kFullS, busy, o);
    if (lane == 0) {
      c.s.dev3n[3 * d + 0] = c.s.peak[d];
      c.s.dev3n[3 * d + 1] = busy;
      c.s.dev3n[3 * d + 2] = makespan - busy;
    }
  }
  if (lane == 0) {
    *c.s.makespan = makespan;
    c.s.xfer4[0] = xcount;
    c.s.xfer4[1] = xbytes;
    c.s.xfer4[2] = dups;
    c.s.xfer4[3] = hits;
    err->status = kOk;
    err->code = E_NONE;
  }
}

// ============================================================================
// K4f — the dataflow simulator: parallel comm mode, every node k > 0.
//
// In parallel mode each (producer i, consumer device d) transfer leaves at
// i's finish and takes comm_time(max bytes over i's consumers on d)
// (simulator.cpp:156-181), so the start of node j, the next entry of its
// device's FIFO, is
//     start_j = max(finish of j's FIFO predecessor,
//                   max over remote parents i of finish_i + c(i, dev j))
// (same-device parents precede j in the FIFO or the run deadlocks, and then
// finish before its predecessor does). Start times are therefore a longest
// path, order-independent: one warp walks each device's FIFO, 32 entries at a
// time, and a lane's entry is ready once every remote parent has published
// its finish; the ready prefix is resolved by a warp max-plus scan
// f_l = max(f_{l-1} + k_l, A_l + k_l). Walkers run in barrier rounds until
// none moves: then either every FIFO is drained or the run is deadlocked
// (the reference's qpos = the walkers' positions).
//
// Memory (simulator.cpp:66-76,121-152): a device's own start/finish events
// alternate in FIFO order; with k > 0 every event pushed at time t is a start
// (finishes at t were pushed earlier), so the heap pops same-time events as
// finish < xfer < start, by node. An output freed at its last consumer's
// finish (GraphStatic) therefore lands before the first start on its device
// at or after that finish time: a bucket per FIFO slot, then one scan per
// device gives the memory at every start, the peak, and the first violation
// (min (t, node) over devices = the heap's first). Zero-duration nodes can
// cascade same-time events out of key order; those problems and sequential
// comm mode stay on the event-loop kernel above.
// ============================================================================
__device__ __forceinline__ int64_t ld_cta(const int64_t *p) {
  int64_t v;
  asm volatile("ld.relaxed.cta.global.s64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_cta(int64_t *p, int64_t v) {
  asm volatile("st.relaxed.cta.global.s64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// K4f prep: grid-wide passes over every problem's nodes and edges
// (blockIdx.y = problem), so a lone large problem uses the whole GPU for them.
// Validation flags and transfer counters go to flow8; out-of-range
// placements are only flagged here (the walker kernel reports them first).
#define BX_SIM_STRIDE(i, N) for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (N); i += gridDim.x * blockDim.x)
constexpr int32_t kNever = 1 << 30;  // rcnt flag: a same-device parent comes later in the FIFO

// K4f takes parallel comm mode; sequential comm with at most 32 devices goes
// through the same passes with the sequencer below in place of the walkers
__device__ __forceinline__ bool flow_ok(const DSim &s) { return s.mode == 1 || (s.mode == 0 && s.n <= 32); }

__device__ __forceinline__ bool flow_skip(const DSim &s) {
  return !flow_ok(s) || s.flow8[0] || s.flow8[1] || s.flow8[2];
}

__global__ void k_sim_prep_a(const DSim *sims, const DGraph *graphs, int base) {
  const DSim s = sims[base + blockIdx.y];
  if (!flow_ok(s)) return;
  const DGraph g = graphs[s.graph];
  const int n = s.n;
  int zero = 0;
  BX_SIM_STRIDE(j, g.V) {
    s.seen[j] = 0;
    s.fin[j] = -1;
    s.bucket[j] = 0;
    s.rcnt[j] = 0;
    if (s.mode == 0) s.ninp[j] = 0;  // sequencer: remote destination mask
    zero |= g.k[j] == 0;
  }
  zero |= s.trace != nullptr;  // record_trace: the event loop records processing order
  if (__syncthreads_or(zero) && threadIdx.x == 0) atomicOr(&s.flow8[0], 1ull);
  BX_SIM_STRIDE(e, g.E) {
    const int i = g.esrc[e], dc = s.device_of[g.edst[e]], di = s.device_of[i];
    if (di != dc && dc >= 0 && dc < n && di >= 0 && di < n) s.mb[static_cast<int64_t>(i) * n + dc] = -1;
  }
}

__global__ void k_sim_prep_b(const DSim *sims, const DGraph *graphs, int base) {
  const DSim s = sims[base + blockIdx.y];
  if (!flow_ok(s)) return;
  const DGraph g = graphs[s.graph];
  const int V = g.V, n = s.n;
  // exec lists (simulator.cpp:84-90): range and device agreement, counts
  int bad = 0;
  const int total = s.exec_off[n];
  BX_SIM_STRIDE(x, total) {
    int lo = 0, hi = n;  // device d with exec_off[d] <= x < exec_off[d+1]
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (s.exec_off[mid] <= x) lo = mid;
      else hi = mid;
    }
    const int m = s.exec_order[x];
    if (m < 0 || m >= V || s.device_of[m] != lo) {
      bad = 1;
    } else {
      atomicAdd(&s.seen[m], 1);
      s.pos[m] = x - s.exec_off[lo];
    }
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&s.flow8[1], 1ull);
  // one transfer per (producer, remote consumer device), max bytes
  unsigned long long cnt = 0, rem = 0;
  BX_SIM_STRIDE(e, g.E) {
    const int i = g.esrc[e], dc = s.device_of[g.edst[e]], di = s.device_of[i];
    uint8_t f = 0;
    if (di != dc && dc >= 0 && dc < n && di >= 0 && di < n) {
      ++rem;
      auto *slot = reinterpret_cast<unsigned long long *>(s.mb + static_cast<int64_t>(i) * n + dc);
      f = atomicCAS(slot, ~0ull, ~0ull - 1) == ~0ull;
      cnt += f;
      if (f && s.mode == 0) atomicOr(reinterpret_cast<unsigned *>(s.ninp + i), 1u << dc);
      // the reference's per-destination slot starts at 0 (simulator.cpp:160-162)
      atomicMax(reinterpret_cast<long long *>(slot), static_cast<long long>(g.ebytes[e] > 0 ? g.ebytes[e] : 0));
    }
    s.first[e] = f;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    cnt += __shfl_xor_sync(kFullS, cnt, o);
    rem += __shfl_xor_sync(kFullS, rem, o);
  }
  if ((threadIdx.x & 31) == 0 && (cnt | rem)) {
    atomicAdd(&s.flow8[3], cnt);
    atomicAdd(&s.flow8[5], rem);
  }
}

__global__ void k_sim_prep_c(const DSim *sims, const DGraph *graphs, int base) {
  const DSim s = sims[base + blockIdx.y];
  if (!flow_ok(s)) return;
  const DGraph g = graphs[s.graph];
  const int V = g.V, n = s.n;
  int bad = 0;
  BX_SIM_STRIDE(j, V) {
    const int d = s.device_of[j];
    if (d < 0 || d >= n || s.seen[j] != 1) bad = 1;
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&s.flow8[2], 1ull);
  unsigned long long by = 0;
  BX_SIM_STRIDE(e, g.E)
  if (s.first[e]) by += s.mb[static_cast<int64_t>(g.esrc[e]) * n + s.device_of[g.edst[e]]];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) by += __shfl_xor_sync(kFullS, by, o);
  if ((threadIdx.x & 31) == 0 && by) atomicAdd(&s.flow8[4], by);
  // per in-CSR slot: the arrival delay on the consumer's device; remote
  // parents counted per consumer, a later same-device parent marks it never
  BX_SIM_STRIDE(x, g.E) {
    const int e = g.in_edge[x];
    const int i = g.esrc[e], c = g.edst[e];
    const int di = s.device_of[i], dc = s.device_of[c];
    if (di < 0 || di >= n || dc < 0 || dc >= n) continue;  // flagged; never walked
    if (di == dc) {
      s.cx[x] = -1;
      if (s.pos[i] >= s.pos[c]) atomicOr(&s.rcnt[c], kNever);
    } else {
      s.cx[x] = comm_time_exact(s.ic, s.pb, s.mb[static_cast<int64_t>(i) * n + dc]);
      atomicAdd(&s.rcnt[c], 1);
    }
  }
}

// remote-parent list offsets in FIFO-slot order (one CTA per problem: a
// block scan over the slots), compute times by slot
__global__ void __launch_bounds__(1024) k_sim_prep_d(const DSim *sims, const DGraph *graphs) {
  __shared__ int wsum[32];
  __shared__ int carry;
  const DSim s = sims[blockIdx.x];
  if (flow_skip(s)) return;
  const DGraph g = graphs[s.graph];
  const int V = g.V;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int b = 0; b < V; b += blockDim.x) {
    const int xs = b + tid;
    int v = 0;
    if (xs < V) {
      const int j = s.exec_order[xs];
      const int rc = s.rcnt[j];
      v = rc & (kNever - 1);
      s.kx[xs] = (rc & kNever) ? -1 : g.k[j];
      s.rcnt[j] = v;  // becomes the fill cursor
    }
    int incl = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int u = __shfl_up_sync(kFullS, incl, o);
      if (lane >= o) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      int w = lane < NW ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int u = __shfl_up_sync(kFullS, w, o);
        if (lane >= o) w += u;
      }
      if (lane < NW) wsum[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    const int before = carry + (warp ? wsum[warp - 1] : 0) + incl - v;
    if (xs < V) s.rp_off[xs] = before;
    __syncthreads();
    if (tid == 0) carry += wsum[NW - 1];
    __syncthreads();
  }
  if (tid == 0) s.rp_off[V] = carry;
}

__global__ void k_sim_prep_e(const DSim *sims, const DGraph *graphs, int base) {
  const DSim s = sims[base + blockIdx.y];
  if (flow_skip(s)) return;
  const DGraph g = graphs[s.graph];
  BX_SIM_STRIDE(x, g.E) {
    const int64_t cc = s.cx[x];
    if (cc < 0) continue;
    const int e = g.in_edge[x];
    if (s.mode == 0 && s.first[e]) {  // the sequencer reads transfer times, not bytes
      const int64_t y = static_cast<int64_t>(g.esrc[e]) * s.n + s.device_of[g.edst[e]];
      s.mb[y] = comm_time_exact(s.ic, s.pb, s.mb[y]);
    }
    const int i = g.esrc[e], c = g.edst[e];
    const int xs = s.exec_off[s.device_of[c]] + s.pos[c];
    const int slot = s.rp_off[xs] + atomicSub(&s.rcnt[c], 1) - 1;
    s.rp_src[slot] = i;
    s.rp_c[slot] = cc;
  }
}

// ---- sequential comm mode: the transfer sequencer ---------------------------
// In sequential mode a finish at t sends its output to each remote consumer
// device in ascending order, each transfer starting at max(t, xfree[src],
// xfree[dst]) and holding both queues (simulator.cpp:163-173), so arrivals
// depend on the global order of finishes. With every k > 0 the heap pops a
// device's start and a transfer's landing no later than anything they cause,
// so the run reduces to a merge of the device FIFOs by (finish, node):
//   * a FIFO head starts at max(finish of its FIFO predecessor, arrival of
//     each remote input on its device) — the last try_start that finds it
//     ready (:113-119); same-device parents finish before its predecessor;
//   * the next finish processed is the minimum (t, node) over the running
//     heads (one per device, lane = device): a head still waiting for an
//     input waits for a finish not yet processed, so its own finish is later;
//   * processing it folds its transfers into the queues (one destination: one
//     max; several: a warp max-plus scan over the destination lanes,
//     X_d = max(X_{d-1}, t, xfree[d]) + c_d), publishes each arrival A(i, d),
//     and wakes a head waiting on exactly that input; the source lane moves
//     to its next FIFO entry.
// mb[i*n + d] holds the transfer time c(i, d) (precomputed in prep_e) until
// i is sent, then -2 - A(i, d): column d is only ever touched by lane d. A
// lane prefetches its next FIFO entry's row into L1.
// Memory, the report and the deadlock verdict are K4f's passes (the starts
// are the same events).
constexpr int kSeqRun = 0, kSeqWait = 1, kSeqDone = 2, kSeqNever = 3;

__device__ __forceinline__ void prefetch_l1(const void *p) { asm volatile("prefetch.global.L1 [%0];" ::"l"(p)); }

__device__ __forceinline__ unsigned long long warp_min_u64s(unsigned long long v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_min_sync(kFullS, hi);
  const unsigned mlo = __reduce_min_sync(kFullS, hi == mhi ? lo : 0xffffffffu);
  return (static_cast<unsigned long long>(mhi) << 32) | mlo;
}

__device__ __forceinline__ void seq_sequencer(const DSim &s) {
  const int n = s.n, lane = threadIdx.x & 31;
  // column `lane` of mb: the transfer time c(p, lane) >= 0 until p is sent,
  // then -2 - A(p, lane) (only lane d ever touches column d)
  int64_t *mc = s.mb + lane;
  // arrival of p's output on this lane's device, -1 while not sent
  auto arrival = [&](int p) -> int64_t {
    const int64_t v = mc[static_cast<int64_t>(p) * n];
    return v >= 0 ? -1 : -2 - v;
  };

  int o = 0, len = 0, pos = 0, st = kSeqDone, h = -1, r = 0, re = 0, cp = -1;
  int64_t prev = 0, xf = 0, ft = 0, amax = 0, kk = 0, mk = 0;
  unsigned hm = 0;
  // FIFO entries pos+1 (n1*) and pos+2 (n2*), loaded ahead of use
  int n1h = -1, n1r = 0, n1re = 0, n2h = -1, n2r = 0, n2re = 0;
  int n1p[4] = {-1, -1, -1, -1};
  unsigned n1m = 0;
  int64_t n1k = 0, n2k = 0;
  auto load2 = [&](int q) {
    if (q < len) {
      const int xs = o + q;
      n2h = s.exec_order[xs];
      n2k = s.kx[xs];
      n2r = s.rp_off[xs];
      n2re = s.rp_off[xs + 1];
    }
  };
  auto shift = [&](int q) {  // entry q (loaded as n2) becomes n1; load q + 1 as n2
    n1h = n2h;
    n1k = n2k;
    n1r = n2r;
    n1re = n2re;
    if (q < len) {
#pragma unroll
      for (int u = 0; u < 4; ++u) n1p[u] = n1r + u < n1re ? s.rp_src[n1r + u] : -1;
      n1m = static_cast<unsigned>(s.ninp[n1h]);
      prefetch_l1(s.mb + static_cast<int64_t>(n1h) * n);  // its transfer times, read when it finishes
    }
    load2(q + 1);
  };
  auto advance = [&](int c0, int c1, int c2, int c3) {  // c_u = rp_src[r + u] where r + u < re
    while (r < re) {
      const int lim = re - r;
      const int64_t v0 = arrival(c0);
      const int64_t v1 = lim > 1 ? arrival(c1) : 0;
      const int64_t v2 = lim > 2 ? arrival(c2) : 0;
      const int64_t v3 = lim > 3 ? arrival(c3) : 0;
      // the first input of the four not sent yet (4: none)
      const int f = v0 < 0 ? 0 : (lim > 1 && v1 < 0) ? 1 : (lim > 2 && v2 < 0) ? 2 : (lim > 3 && v3 < 0) ? 3 : 4;
      const int take = min(f, lim);
      if (take > 0) amax = smax(amax, v0);
      if (take > 1) amax = smax(amax, v1);
      if (take > 2) amax = smax(amax, v2);
      if (take > 3) amax = smax(amax, v3);
      r += take;
      if (f < 4) {  // waits for this input (f < 4 only within the chunk)
        cp = f == 0 ? c0 : f == 1 ? c1 : f == 2 ? c2 : c3;
        return;
      }
      if (r >= re) break;
      c0 = s.rp_src[r];
      c1 = r + 1 < re ? s.rp_src[r + 1] : -1;
      c2 = r + 2 < re ? s.rp_src[r + 2] : -1;
      c3 = r + 3 < re ? s.rp_src[r + 3] : -1;
    }
    st = kSeqRun;
    ft = amax + kk;
    s.sx[o + pos] = amax;
    s.start[h] = amax;
  };
  auto setup = [&]() {  // entry pos becomes the head
    if (pos >= len) {
      st = kSeqDone;
      return;
    }
    h = n1h;
    kk = n1k;
    r = n1r;
    re = n1re;
    hm = n1m;
    const int p0 = n1p[0], p1 = n1p[1], p2 = n1p[2], p3 = n1p[3];
    amax = prev;
    shift(pos + 1);
    if (kk < 0) {  // a same-device parent comes later in the FIFO: never ready
      st = kSeqNever;
      return;
    }
    st = kSeqWait;
    advance(p0, p1, p2, p3);
  };
  if (lane < n) {
    o = s.exec_off[lane];
    len = s.exec_off[lane + 1] - o;
    load2(0);
    shift(0);
    setup();
  }
  while (true) {
    const bool run = st == kSeqRun;
    if (!__any_sync(kFullS, run)) break;
    // the next finish: minimum (t, node) over the running heads
    const unsigned long long mt = warp_min_u64s(run ? static_cast<unsigned long long>(ft) : ~0ull);
    const bool tied = run && static_cast<unsigned long long>(ft) == mt;
    const unsigned tie = __ballot_sync(kFullS, tied);
    int w = __ffs(tie) - 1;
    if (tie & (tie - 1)) {
      const unsigned hn = __reduce_min_sync(kFullS, tied ? static_cast<unsigned>(h) : 0xffffffffu);
      w = __ffs(__ballot_sync(kFullS, tied && static_cast<unsigned>(h) == hn)) - 1;
    }
    const int64_t t = static_cast<int64_t>(mt);
    const int i = __shfl_sync(kFullS, h, w);
    const unsigned M = __shfl_sync(kFullS, hm, w);
    if (M) {
      const int64_t x0 = __shfl_sync(kFullS, xf, w);
      const bool dst = (M >> lane) & 1u;
      int64_t X = 0;  // the queues' free time after this lane's transfer
      int64_t xl;     // the source queue's afterwards
      if (!(M & (M - 1))) {  // one destination
        if (dst) X = smax(smax(x0, t), xf) + mc[static_cast<int64_t>(i) * n];
        xl = __shfl_sync(kFullS, X, __ffs(M) - 1);
      } else {
        int64_t a = 0, b = INT64_MIN / 4;  // identity of f(X) = max(X + a, b)
        if (dst) {
          const int64_t c = mc[static_cast<int64_t>(i) * n];
          a = c;
          b = smax(t, xf) + c;
        }
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int64_t a2 = __shfl_up_sync(kFullS, a, off), b2 = __shfl_up_sync(kFullS, b, off);
          if (lane >= off) {
            b = smax(b2 + a, b);
            a = a2 + a;
          }
        }
        X = smax(x0 + a, b);
        xl = __shfl_sync(kFullS, X, 31);
      }
      if (dst) {
        xf = X;
        mc[static_cast<int64_t>(i) * n] = -2 - X;
        if (st == kSeqWait && cp == i) {
          amax = smax(amax, X);
          ++r;
          advance(r < re ? s.rp_src[r] : -1, r + 1 < re ? s.rp_src[r + 1] : -1, r + 2 < re ? s.rp_src[r + 2] : -1,
                  r + 3 < re ? s.rp_src[r + 3] : -1);
        }
      }
      if (lane == w) xf = xl;
    }
    if (lane == w) {
      s.fin[i] = t;
      prev = t;
      mk = smax(mk, t);
      ++pos;
      setup();
    }
  }
  if (lane < n) s.qpos[lane] = pos;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) mk = smax(mk, __shfl_xor_sync(kFullS, mk, off));
  if (lane == 0) *s.makespan = mk;
}

constexpr int kWalkSpin = 64;

// validation verdicts and permanent memory, shared by the walkers and the
// sequencer; false when the run already ended (error set)
__device__ bool flow_preamble(const DSim &s, const DGraph &g, int *sh_bad) {
  const int n = s.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  DErr *err = s.err;
  // validate_placement (simulator.cpp:78-97), decided by its first failing check
  if (s.flow8[1] || s.flow8[2]) {
    if (tid == 0) {
      err->status = kValidation;
      err->code = s.flow8[1] ? E_SIM_EXEC : E_SIM_ONCE;
    }
    return false;
  }
  if (tid == 0) *sh_bad = INT32_MAX;
  __syncthreads();
  // permanent memory up front, device by device in FIFO order (:209-214)
  for (int d = warp; d < n; d += NW) {
    const int o = s.exec_off[d], len = s.exec_off[d + 1] - o;
    const int64_t cap = s.cap[d];
    int64_t run = 0;
    int vbad = INT32_MAX;
    int64_t vmem = 0;
    for (int b = 0; b < len; b += 32) {
      const int p = b + lane;
      int64_t v = p < len ? g.perm[s.exec_order[o + p]] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        int64_t u = __shfl_up_sync(kFullS, v, off);
        if (lane >= off) v += u;
      }
      const int64_t m = run + v;
      unsigned over = __ballot_sync(kFullS, p < len && m > cap);
      if (over && vbad == INT32_MAX) {
        const int l = __ffs(over) - 1;
        vbad = b + l;
        vmem = __shfl_sync(kFullS, m, l);
      }
      run = __shfl_sync(kFullS, m, 31);
    }
    if (lane == 0) {
      s.mem[d] = run;
      s.qpos[d] = 0;
      s.xfree[d] = 0;
      s.dest_cnt[d] = vbad;  // first violating FIFO slot (perm)
      s.dest_bytes[d] = vmem;
      if (vbad != INT32_MAX) atomicMin(sh_bad, d);
    }
  }
  __syncthreads();
  if (*sh_bad != INT32_MAX) {
    if (tid == 0) {
      const int d = *sh_bad;
      err->status = kInfeasible;
      err->code = E_SIM_MEMORY;
      err->a = d;
      err->b = 0;
      err->c = s.exec_order[s.exec_off[d] + s.dest_cnt[d]];
      err->d = s.dest_bytes[d];
    }
    return false;
  }
  return true;
}

// sequential comm mode, <= 32 devices: warp 0 sequences, warp 1 warms L1
// sequential comm mode, <= 32 devices: one warp per problem
__global__ void __launch_bounds__(32, 1) k_sim_seq(const DSim *sims, int nsims, const DGraph *graphs) {
  __shared__ int sh_bad;
  const DSim s = sims[blockIdx.x];
  if (s.mode != 0 || s.n > 32 || s.flow8[0]) return;  // zero-duration nodes, traces: event loop
  const DGraph g = graphs[s.graph];
  if (!flow_preamble(s, g, &sh_bad)) return;
  seq_sequencer(s);
}

// K4f walkers: validation verdicts, permanent memory, then the FIFO walk.
__global__ void __launch_bounds__(1024) k_sim_flow(const DSim *sims, int nsims, const DGraph *graphs) {
  __shared__ long long sh_mk;
  __shared__ int sh_bad;
  const DSim s = sims[blockIdx.x];
  if (s.mode != 1) return;
  const DGraph g = graphs[s.graph];
  const int n = s.n;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  if (s.flow8[0]) return;  // zero-duration nodes: event-loop kernel
  if (tid == 0) sh_mk = 0;
  if (!flow_preamble(s, g, &sh_bad)) return;

  // ---- walkers ----------------------------------------------------------------
  int64_t mk = 0;
  while (true) {
    int adv = 0;
    for (int d = warp; d < n; d += NW) {
      const int o = s.exec_off[d], len = s.exec_off[d + 1] - o;
      int p = s.qpos[d];
      int64_t prev = s.xfree[d];
      int spins = 0;
      while (p < len) {
        const int idx = p + lane, xs = o + idx;
        bool ok = false;
        int64_t A = 0, kk = 0;
        int j = -1;
        if (idx < len) {
          kk = s.kx[xs];
          j = s.exec_order[xs];
          int r = s.rp_off[xs];
          const int re = s.rp_off[xs + 1];
          ok = kk >= 0;
          for (; ok && r + 1 < re; r += 2) {  // two remote parents per step
            const int i0 = s.rp_src[r], i1 = s.rp_src[r + 1];
            const int64_t c0 = s.rp_c[r], c1 = s.rp_c[r + 1];
            const int64_t f0 = ld_cta(s.fin + i0), f1 = ld_cta(s.fin + i1);
            ok = f0 >= 0 && f1 >= 0;
            A = smax(A, smax(f0 + c0, f1 + c1));
          }
          if (ok && r < re) {
            const int64_t f0 = ld_cta(s.fin + s.rp_src[r]);
            ok = f0 >= 0;
            A = smax(A, f0 + s.rp_c[r]);
          }
        }
        const unsigned okm = __ballot_sync(kFullS, ok);
        const int L = okm == kFullS ? 32 : __ffs(~okm) - 1;
        if (L == 0) {
          // the other walkers of this CTA publish as they go: poll a while
          // before ending the round (fewer barrier rounds; exactness never
          // depends on it, the barrier round decides termination)
          if (++spins <= kWalkSpin) {
            __nanosleep(200);
            continue;
          }
          break;
        }
        spins = 0;
        int64_t al = kk, be = A + kk;  // g_l(f) = max(f + al, be), composed over lanes <= l
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int64_t a2 = __shfl_up_sync(kFullS, al, off), b2 = __shfl_up_sync(kFullS, be, off);
          if (lane >= off) {
            be = smax(b2 + al, be);
            al = a2 + al;
          }
        }
        const int64_t f = smax(prev + al, be);
        if (lane < L) {
          s.sx[xs] = f - kk;
          s.start[j] = f - kk;
          st_cta(s.fin + j, f);
        }
        prev = __shfl_sync(kFullS, f, L - 1);
        p += L;
        adv = 1;
        if (L < 32) break;
      }
      if (lane == 0) {
        s.qpos[d] = p;
        s.xfree[d] = prev;
      }
      mk = smax(mk, prev);
    }
    if (!__syncthreads_or(adv)) break;
  }
  if (lane == 0) atomicMax(&sh_mk, static_cast<long long>(mk));
  __syncthreads();
  if (tid == 0) *s.makespan = sh_mk;
}

// GraphStatic: an output is freed at its last consumer's finish, before the
// first start on its device at or after that time (grid-wide).
__global__ void k_sim_free(const DSim *sims, const DGraph *graphs, int base) {
  const DSim s = sims[base + blockIdx.y];
  if (flow_skip(s) || s.mem_mode != 0 || s.err->status) return;
  const DGraph g = graphs[s.graph];
  BX_SIM_STRIDE(i, g.V) {
    const int b = g.out_off[i], e = g.out_off[i + 1];
    if (b == e) continue;  // freed at its own finish
    int64_t lt = -1;
    int lc = -1;
    bool all = true;
    for (int y = b; y < e; ++y) {
      const int c = g.edst[y];
      const int64_t f = s.fin[c];
      if (f < 0) {
        all = false;
        break;
      }
      if (f > lt || (f == lt && c > lc)) {
        lt = f;
        lc = c;
      }
    }
    if (!all) continue;
    const int d = s.device_of[i], o = s.exec_off[d], started = s.qpos[d];
    int lo = 0, hi = started;  // first started slot with start >= lt
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (s.sx[o + mid] >= lt) hi = mid;
      else lo = mid + 1;
    }
    if (lo < started)
      atomicAdd(reinterpret_cast<unsigned long long *>(s.bucket + o + lo), static_cast<unsigned long long>(g.outb[i]));
  }
}

// memory at every start of one device (CTA per (device, problem)): block
// scans over the started FIFO slots; peak, first violation, busy time.
__global__ void __launch_bounds__(1024) k_sim_mem(const DSim *sims, const DGraph *graphs, int base) {
  __shared__ long long wsum[32];
  __shared__ long long s_carry, s_peak, s_busy, s_vm;
  __shared__ int s_vp, s_vj;
  const DSim s = sims[base + blockIdx.y];
  const int d = blockIdx.x;
  if (d >= s.n || flow_skip(s) || s.err->status) return;
  const DGraph g = graphs[s.graph];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, NW = blockDim.x >> 5;
  const int o = s.exec_off[d], started = s.qpos[d];
  const int64_t cap = s.cap[d];
  if (tid == 0) {
    s_carry = s.mem[d];
    s_peak = s.mem[d];
    s_busy = 0;
    s_vp = INT32_MAX;
  }
  __syncthreads();
  int64_t peak = 0, busy = 0;
  for (int b = 0; b < started; b += blockDim.x) {
    const int p = b + tid;
    int64_t ch = 0, w = 0, fr = 0;
    int j = -1;
    if (p < started) {
      j = s.exec_order[o + p];
      const int64_t tmp = g.temp[j], out = g.outb[j];
      ch = tmp + out;
      const bool drop = s.mem_mode == 0 && g.out_off[j + 1] == g.out_off[j];
      fr = s.bucket[o + p];
      w = ch - tmp - (drop ? out : 0) - fr;
      busy += g.k[j];
    }
    long long incl = w;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      const long long u = __shfl_up_sync(kFullS, incl, off);
      if (lane >= off) incl += u;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      long long x = lane < NW ? wsum[lane] : 0;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const long long u = __shfl_up_sync(kFullS, x, off);
        if (lane >= off) x += u;
      }
      if (lane < NW) wsum[lane] = x;
    }
    __syncthreads();
    const int64_t m = s_carry + (warp ? wsum[warp - 1] : 0) + (incl - w) - fr + ch;
    if (p < started) {
      peak = smax(peak, m);
      if (m > cap) atomicMin(&s_vp, p);
    }
    __syncthreads();
    if (p == s_vp) {  // the run stops at its first violation
      s_vm = m;
      s_vj = j;
    }
    if (tid == 0) s_carry += wsum[NW - 1];
    const bool stop = s_vp != INT32_MAX;
    __syncthreads();
    if (stop) break;
  }
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    peak = smax(peak, __shfl_xor_sync(kFullS, peak, off));
    busy += __shfl_xor_sync(kFullS, busy, off);
  }
  if (lane == 0) {
    atomicMax(&s_peak, static_cast<long long>(peak));
    atomicAdd(reinterpret_cast<unsigned long long *>(&s_busy), static_cast<unsigned long long>(busy));
  }
  __syncthreads();
  if (tid != 0) return;
  s.dv[4 * d + 0] = s_peak;
  s.dev3n[3 * d + 1] = s_busy;
  if (s_vp == INT32_MAX) {
    s.dv[4 * d + 1] = INT64_MAX;
    return;
  }
  s.dv[4 * d + 1] = s.sx[o + s_vp];
  s.dv[4 * d + 2] = s_vj;
  s.dv[4 * d + 3] = s_vm;
}

// the verdict: first violation (min (t, node) over devices), deadlock, or the report
__global__ void k_sim_report(const DSim *sims, int nsims) {
  const int sid = blockIdx.x * blockDim.x + threadIdx.x;
  if (sid >= nsims) return;
  const DSim s = sims[sid];
  if (flow_skip(s) || s.err->status) return;
  DErr *err = s.err;
  const int n = s.n;
  int vd = -1;
  for (int d = 0; d < n; ++d) {
    const int64_t t = s.dv[4 * d + 1];
    if (t == INT64_MAX) continue;
    if (vd < 0 || t < s.dv[4 * vd + 1] || (t == s.dv[4 * vd + 1] && s.dv[4 * d + 2] < s.dv[4 * vd + 2])) vd = d;
  }
  if (vd >= 0) {
    err->status = kInfeasible;
    err->code = E_SIM_MEMORY;
    err->a = vd;
    err->b = s.dv[4 * vd + 1];
    err->c = s.dv[4 * vd + 2];
    err->d = s.dv[4 * vd + 3];
    return;
  }
  for (int d = 0; d < n; ++d) {
    if (s.qpos[d] < s.exec_off[d + 1] - s.exec_off[d]) {  // deadlock (:234-246)
      err->status = kValidation;
      err->code = E_SIM_DEADLOCK;
      err->a = d;
      err->c = s.exec_order[s.exec_off[d] + s.qpos[d]];
      return;
    }
  }
  const int64_t makespan = *s.makespan;
  for (int d = 0; d < n; ++d) {
    s.dev3n[3 * d + 0] = s.dv[4 * d + 0];
    s.dev3n[3 * d + 2] = makespan - s.dev3n[3 * d + 1];
  }
  s.xfer4[0] = static_cast<int64_t>(s.flow8[3]);
  s.xfer4[1] = static_cast<int64_t>(s.flow8[4]);
  s.xfer4[2] = 0;  // a tensor is sent once per device: duplicates never arise
  s.xfer4[3] = static_cast<int64_t>(s.flow8[5] - s.flow8[3]);
  err->status = kOk;
  err->code = E_NONE;
}

void launch_simulate(const DSim *sims, int nsims, const DGraph *graphs, int maxn, int force_cap, cudaStream_t s) {
  // K4f: grid-wide passes (blockIdx.y = problem), then one CTA per problem
  // for the walkers, per device for the memory scans; K4 takes the problems
  // K4f leaves (sequential comm, zero-duration nodes) after the first pass
  const unsigned gx = nsims <= 16 ? 148 : nsims <= 148 ? 16 : 2;
  auto grid = [&](auto kern, unsigned x, int threads) {
    for (int b = 0; b < nsims; b += 65535) {
      const dim3 g(x, static_cast<unsigned>(nsims - b < 65535 ? nsims - b : 65535));
      kern<<<g, threads, 0, s>>>(sims, graphs, b);
    }
  };
  grid(k_sim_prep_a, gx, 256);
  // force_cap >= 0 (bx_plan_options.sim_heap_cap, tests): a tiny shared-memory
  // heap exercises the spill to global memory
  // per-device state goes to shared memory when it fits beside the heaps
  constexpr size_t kSmemBudget = 200 * 1024;
  int dev_slots = maxn;
  if (6 * sizeof(int64_t) * size_t(dev_slots) * 4 + 2 * sizeof(int64_t) * 1024 * 4 > kSmemBudget) dev_slots = 0;
  const size_t dev_bytes = 6 * sizeof(int64_t) * static_cast<size_t>(dev_slots);
  if (force_cap >= 0) {
    const size_t sm = 2 * sizeof(int64_t) * static_cast<size_t>(force_cap) + dev_bytes;
    cudaFuncSetAttribute(k_simulate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    k_simulate<1><<<nsims, 32, sm, s>>>(sims, nsims, graphs, force_cap, dev_slots);
  } else if (nsims <= 148) {  // a few problems: one per CTA, a 12k-event shared-memory heap each
    const int kCap = static_cast<int>(std::min<size_t>(12288, (kSmemBudget - dev_bytes) / (2 * sizeof(int64_t))));
    const size_t sm = 2 * sizeof(int64_t) * kCap + dev_bytes;
    cudaFuncSetAttribute(k_simulate<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    k_simulate<1><<<nsims, 32, sm, s>>>(sims, nsims, graphs, kCap, dev_slots);
  } else {
    constexpr int W = 4, kCap = 1024;
    const size_t sm = (2 * sizeof(int64_t) * kCap + dev_bytes) * W;
    cudaFuncSetAttribute(k_simulate<W>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    k_simulate<W><<<(nsims + W - 1) / W, 32 * W, sm, s>>>(sims, nsims, graphs, kCap, dev_slots);
  }
  grid(k_sim_prep_b, gx, 256);
  grid(k_sim_prep_c, gx, 256);
  const int cta = nsims <= 148 ? 1024 : 256;
  k_sim_prep_d<<<nsims, cta, 0, s>>>(sims, graphs);
  grid(k_sim_prep_e, gx, 256);
  k_sim_flow<<<nsims, cta, 0, s>>>(sims, nsims, graphs);
  k_sim_seq<<<nsims, 32, 0, s>>>(sims, nsims, graphs);
  grid(k_sim_free, gx, 256);
  grid(k_sim_mem, static_cast<unsigned>(maxn), cta);
  k_sim_report<<<(nsims + 127) / 128, 128, 0, s>>>(sims, nsims);
}

// ---------------------------------------------------------------- K3 ----
// round_and_extract (lp.cpp:280-326). Candidates are edges with x < thr
// (NaN never qualifies). Per source keep the lexicographic min (x, dst);
// then, among the kept edges, per destination keep the min (x, src).
// Both are segmented lexicographic minima done edge-parallel with 64-bit
// atomics in two passes each: first the minimum x (as an order-preserving
// integer image, -0.0 folded onto +0.0 like the double compare does), then
// the minimum peer index among the edges that attain it. No edge order is
// assumed; ties cannot survive both passes because (src, dst) is unique.
__device__ __forceinline__ unsigned long long order_bits(double x) {
  if (x == 0.0) x = 0.0;
  unsigned long long u = static_cast<unsigned long long>(__double_as_longlong(x));
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}


#define BX_GRID_STRIDE(i, N) for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < (N); i += gridDim.x * blockDim.x)

__global__ void k_x_src_min(XCtx c) {
  BX_GRID_STRIDE(e, c.E) {
    double v = c.x[e];
    if (!(v < c.thr)) continue;
    int s = c.esrc[e];
    atomicMin(&c.src_min[s], order_bits(v));
    atomicAdd(&c.cnt_src[s], 1);
  }
}
__global__ void k_x_src_peer(XCtx c) {
  BX_GRID_STRIDE(e, c.E) {
    double v = c.x[e];
    if (!(v < c.thr)) continue;
    int s = c.esrc[e];
    if (order_bits(v) == c.src_min[s]) atomicMin(&c.src_peer[s], c.edst[e]);
  }
}
__global__ void k_x_src_pick(XCtx c) {
  BX_GRID_STRIDE(e, c.E) {
    double v = c.x[e];
    if (!(v < c.thr)) continue;
    int s = c.esrc[e];
    if (order_bits(v) == c.src_min[s] && c.edst[e] == c.src_peer[s]) c.best_edge[s] = e;
  }
}
__global__ void k_x_dst_min(XCtx c) {
  BX_GRID_STRIDE(i, c.V) {
    int e = c.best_edge[i];
    if (e < 0) continue;
    int d = c.edst[e];
    atomicMin(&c.dst_min[d], order_bits(c.x[e]));
    atomicAdd(&c.cnt_dst[d], 1);
  }
}
__global__ void k_x_dst_peer(XCtx c) {
  BX_GRID_STRIDE(i, c.V) {
    int e = c.best_edge[i];
    if (e < 0) continue;
    int d = c.edst[e];
    if (order_bits(c.x[e]) == c.dst_min[d]) atomicMin(&c.dst_peer[d], i);
  }
}
__global__ void k_x_finish(XCtx c) {
  int fav = 0, rep = 0;
  BX_GRID_STRIDE(i, c.V) {
    if (c.cnt_src[i] > 1) ++rep;
    if (c.cnt_dst[i] > 1) ++rep;
    if (c.cnt_dst[i] > 0) {
      int s = c.dst_peer[i];
      c.fav_parent[i] = s;
      c.fav_child[s] = i;  // a source keeps at most one edge: no race
      ++fav;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fav += __shfl_xor_sync(kFullS, fav, o);
    rep += __shfl_xor_sync(kFullS, rep, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&c.stats2[0], fav);
    atomicAdd(&c.stats2[1], rep);
  }
}

void launch_extract(const XCtx &c, cudaStream_t s) {
  auto grid = [](int N) {
    int nb = (N + 255) / 256;
    return nb < 1 ? 1 : (nb > 1184 ? 1184 : nb);
  };
  k_x_src_min<<<grid(c.E), 256, 0, s>>>(c);
  k_x_src_peer<<<grid(c.E), 256, 0, s>>>(c);
  k_x_src_pick<<<grid(c.E), 256, 0, s>>>(c);
  k_x_dst_min<<<grid(c.V), 256, 0, s>>>(c);
  k_x_dst_peer<<<grid(c.V), 256, 0, s>>>(c);
  k_x_finish<<<grid(c.V), 256, 0, s>>>(c);
}

}  // namespace bx

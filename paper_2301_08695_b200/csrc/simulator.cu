// K4 — the event-driven makespan simulator (simulate, proj/src/simulator.cpp
// :26-278) and K3 — favourite-child extraction (round_and_extract,
// proj/src/lp.cpp:280-326), for sm_100a.
//
// K4: one warp per (graph, placement) problem. Events are processed in the
// reference's heap order (t, kind{finish 0 < xfer_done 1 < start 2}, a, b)
// (simulator.cpp:14-24); the heap stores (t, packed(kind, a, b)) pairs so one
// 128-bit compare orders them. Lane 0 owns the heap; the whole warp scans
// in/out-edge lists (inputs_resident, the per-destination max-bytes map)
// and the per-device tables.
#include "bx_device.cuh"

namespace bx {

constexpr unsigned kFullS = 0xffffffffu;

__device__ __forceinline__ int64_t smax(int64_t a, int64_t b) { return a > b ? a : b; }

// packed = kind << 58 | a << 20 | b   (a < 2^38, b < 2^20)
__device__ __forceinline__ int64_t pack_ev(int kind, int a, int b) {
  return (static_cast<int64_t>(kind) << 58) | (static_cast<int64_t>(a) << 20) | static_cast<int64_t>(b);
}

struct Heap {
  int64_t *t, *k;
  int64_t size;
  __device__ bool less(int64_t x, int64_t y) const { return t[x] < t[y] || (t[x] == t[y] && k[x] < k[y]); }
  __device__ void swap(int64_t x, int64_t y) {
    int64_t a = t[x], b = k[x];
    t[x] = t[y];
    k[x] = k[y];
    t[y] = a;
    k[y] = b;
  }
  __device__ void push(int64_t tt, int64_t kk) {
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

// inputs_resident (simulator.cpp:100-111), warp-cooperative.
__device__ bool inputs_resident(const SimCtx &c, int j) {
  int dev = c.s.device_of[j];
  bool ok = true;
  for (int x = c.g.in_off[j] + c.lane; x < c.g.in_off[j + 1]; x += 32) {
    int i = c.g.esrc[c.g.in_edge[x]];
    if (!c.s.finished[i]) ok = false;
    else if (c.s.device_of[i] != dev && !c.s.resident[static_cast<int64_t>(i) * c.n + dev]) ok = false;
  }
  return __all_sync(kFullS, ok);
}

// try_start (simulator.cpp:113-119). Warp-uniform control flow; lane 0 pushes.
__device__ void try_start(SimCtx &c, int dev, int64_t now) {
  if (c.s.busy[dev]) return;
  int len = c.s.exec_off[dev + 1] - c.s.exec_off[dev];
  int q = c.s.qpos[dev];
  if (q >= len) return;
  int j = c.s.exec_order[c.s.exec_off[dev] + q];
  if (c.s.start_q[j]) return;
  if (!inputs_resident(c, j)) return;
  __syncwarp();
  if (c.lane == 0) {
    c.s.start_q[j] = 1;
    c.h.push(now, pack_ev(2, j, 0));
  }
  c.h.size = __shfl_sync(kFullS, c.h.size, 0);
  __syncwarp();
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
__global__ void __launch_bounds__(32 * kWarps) k_simulate(const DSim *sims, int nsims, const DGraph *graphs) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sid = blockIdx.x * kWarps + warp;
  if (sid >= nsims) return;
  SimCtx c;
  c.s = sims[sid];
  c.g = graphs[c.s.graph];
  c.V = c.g.V;
  c.n = c.s.n;
  c.lane = lane;
  if (c.s.mode == 1) {
    // parallel comm mode without zero-duration nodes belongs to K4f
    bool zero = false;
    for (int j = lane; j < c.V; j += 32) zero |= c.g.k[j] == 0;
    if (!__any_sync(kFullS, zero)) return;
  }
  c.h.t = c.s.heap_t;
  c.h.k = c.s.heap_k;
  c.h.size = 0;
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
        c.s.busy[dev] = 0;
        c.s.qpos[dev]++;
        c.s.finished[j] = 1;
        c.s.mem[dev] -= c.g.temp[j];
        if (c.s.mem_mode == 0) {
          if (c.s.consumers_left[j] == 0) c.s.mem[dev] -= c.g.outb[j];
          for (int x = c.g.in_off[j]; x < c.g.in_off[j + 1]; ++x) {
            int i = c.g.esrc[c.g.in_edge[x]];
            if (--c.s.consumers_left[i] == 0) c.s.mem[c.s.device_of[i]] -= c.g.outb[i];
          }
        }
      }
      __syncwarp();
      // destinations: max bytes per remote consumer device
      int remote = 0;
      for (int y = c.g.out_off[j] + lane; y < c.g.out_off[j + 1]; y += 32) {
        int cdev = c.s.device_of[c.g.edst[y]];
        if (cdev == dev) continue;
        ++remote;
        c.s.dest_cnt[cdev] = 1;
        atomicMax(reinterpret_cast<unsigned long long *>(&c.s.dest_bytes[cdev]),
                  static_cast<unsigned long long>(c.g.ebytes[y]));
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
          c.h.push(begin + cc, pack_ev(1, j, cdev));
        }
      }
      distinct = __shfl_sync(kFullS, distinct, 0);
      hits += remote - distinct;
      c.h.size = __shfl_sync(kFullS, c.h.size, 0);
      __syncwarp();
      try_start(c, dev, t);
    } else {
      // run_xfer_done (:186-190)
      if (lane == 0) c.s.resident[static_cast<int64_t>(a) * n + b] = 1;
      __syncwarp();
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

__global__ void __launch_bounds__(1024) k_sim_flow(const DSim *sims, int nsims, const DGraph *graphs) {
  __shared__ unsigned long long sh_x[3];  // transfers, bytes, remote edges
  __shared__ long long sh_mk;
  __shared__ int sh_bad;
  const DSim s = sims[blockIdx.x];
  if (s.mode != 1) return;
  const DGraph g = graphs[s.graph];
  const int V = g.V, E = g.E, n = s.n;
  const int tid = threadIdx.x, NT = blockDim.x, lane = tid & 31, warp = tid >> 5, NW = NT >> 5;
  DErr *err = s.err;
  int zero = 0;
  for (int j = tid; j < V; j += NT) zero |= g.k[j] == 0;
  if (__syncthreads_or(zero)) return;  // event-loop kernel

  // ---- validate_placement (simulator.cpp:78-97) ------------------------------
  for (int j = tid; j < V; j += NT) s.seen[j] = 0;
  if (tid == 0) {
    sh_x[0] = sh_x[1] = sh_x[2] = 0;
    sh_mk = 0;
    sh_bad = INT32_MAX;
  }
  __syncthreads();
  int bad = 0;
  for (int d = 0; d < n; ++d) {
    const int o = s.exec_off[d], e = s.exec_off[d + 1];
    for (int x = o + tid; x < e; x += NT) {
      const int m = s.exec_order[x];
      if (m < 0 || m >= V || s.device_of[m] != d) {
        bad = 1;
      } else {
        atomicAdd(&s.seen[m], 1);
        s.pos[m] = x - o;
      }
    }
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) {
      err->status = kValidation;
      err->code = E_SIM_EXEC;
    }
    return;
  }
  for (int j = tid; j < V; j += NT) {
    const int d = s.device_of[j];
    if (d < 0 || d >= n || s.seen[j] != 1) bad = 1;
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) {
      err->status = kValidation;
      err->code = E_SIM_ONCE;
    }
    return;
  }

  // ---- transfers: one per (producer, remote consumer device), max bytes ------
  for (int j = tid; j < V; j += NT) {
    s.fin[j] = -1;
    s.bucket[j] = 0;
  }
  for (int e = tid; e < E; e += NT) {
    const int i = g.esrc[e], dc = s.device_of[g.edst[e]];
    if (s.device_of[i] != dc) s.mb[static_cast<int64_t>(i) * n + dc] = -1;
  }
  __syncthreads();
  {
    unsigned long long cnt = 0, rem = 0;
    for (int e = tid; e < E; e += NT) {
      const int i = g.esrc[e], dc = s.device_of[g.edst[e]];
      uint8_t f = 0;
      if (s.device_of[i] != dc) {
        ++rem;
        auto *slot = reinterpret_cast<unsigned long long *>(s.mb + static_cast<int64_t>(i) * n + dc);
        f = atomicCAS(slot, ~0ull, ~0ull - 1) == ~0ull;
        cnt += f;
        atomicMax(reinterpret_cast<long long *>(slot), static_cast<long long>(g.ebytes[e]));
      }
      s.first[e] = f;
    }
    atomicAdd(&sh_x[0], cnt);
    atomicAdd(&sh_x[2], rem);
  }
  __syncthreads();
  {
    unsigned long long by = 0;
    for (int e = tid; e < E; e += NT)
      if (s.first[e]) by += s.mb[static_cast<int64_t>(g.esrc[e]) * n + s.device_of[g.edst[e]]];
    atomicAdd(&sh_x[1], by);
  }
  // per in-CSR slot: the parent and its arrival delay on the consumer's device
  for (int x = tid; x < E; x += NT) {
    const int e = g.in_edge[x];
    const int i = g.esrc[e], c = g.edst[e];
    const int di = s.device_of[i], dc = s.device_of[c];
    s.psrc[x] = i;
    s.cx[x] = di == dc ? (s.pos[i] < s.pos[c] ? -1 : -2)
                       : comm_time_exact(s.ic, s.pb, s.mb[static_cast<int64_t>(i) * n + dc]);
  }
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
      if (vbad != INT32_MAX) atomicMin(&sh_bad, d);
    }
  }
  __syncthreads();
  if (sh_bad != INT32_MAX) {
    if (tid == 0) {
      const int d = sh_bad;
      err->status = kInfeasible;
      err->code = E_SIM_MEMORY;
      err->a = d;
      err->b = 0;
      err->c = s.exec_order[s.exec_off[d] + s.dest_cnt[d]];
      err->d = s.dest_bytes[d];
    }
    return;
  }

  // ---- walkers ----------------------------------------------------------------
  int64_t mk = 0;
  while (true) {
    int adv = 0;
    for (int d = warp; d < n; d += NW) {
      const int o = s.exec_off[d], len = s.exec_off[d + 1] - o;
      int p = s.qpos[d];
      int64_t prev = s.xfree[d];
      while (p < len) {
        const int idx = p + lane;
        bool ok = false;
        int64_t A = 0, kk = 0;
        int j = -1;
        if (idx < len) {
          j = s.exec_order[o + idx];
          kk = g.k[j];
          ok = true;
          const int xe = g.in_off[j + 1];
          for (int x = g.in_off[j]; x < xe; ++x) {
            const int64_t cc = s.cx[x];
            if (cc == -1) continue;
            if (cc == -2) {
              ok = false;
              break;
            }
            const int64_t f = ld_cta(s.fin + s.psrc[x]);
            if (f < 0) {
              ok = false;
              break;
            }
            A = smax(A, f + cc);
          }
        }
        const unsigned okm = __ballot_sync(kFullS, ok);
        const int L = okm == kFullS ? 32 : __ffs(~okm) - 1;
        if (L == 0) break;
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
          s.sx[o + idx] = f - kk;
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

  // ---- memory at every start ------------------------------------------------------
  if (s.mem_mode == 0) {
    for (int i = tid; i < V; i += NT) {
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
      const int d = s.device_of[i], o = s.exec_off[d];
      int lo = 0, hi = s.qpos[d];  // first started slot with start >= lt
      while (lo < hi) {
        const int mid = (lo + hi) >> 1;
        if (s.sx[o + mid] >= lt) hi = mid;
        else lo = mid + 1;
      }
      if (lo < s.qpos[d]) atomicAdd(reinterpret_cast<unsigned long long *>(s.bucket + o + lo),
                                    static_cast<unsigned long long>(g.outb[i]));
    }
  }
  __syncthreads();
  for (int d = warp; d < n; d += NW) {
    const int o = s.exec_off[d], started = s.qpos[d];
    const int64_t cap = s.cap[d];
    int64_t run = s.mem[d], peak = run, vt = INT64_MAX, vm = 0;
    int vj = INT32_MAX;
    int64_t busy = 0;
    for (int b = 0; b < started; b += 32) {
      const int p = b + lane;
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
      int64_t incl = w;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int64_t u = __shfl_up_sync(kFullS, incl, off);
        if (lane >= off) incl += u;
      }
      const int64_t m = run + (incl - w) - fr + ch;
      if (p < started) peak = smax(peak, m);
      const unsigned over = __ballot_sync(kFullS, p < started && m > cap);
      if (over && vt == INT64_MAX) {
        const int l = __ffs(over) - 1;
        vt = s.sx[o + b + l];
        vj = __shfl_sync(kFullS, j, l);
        vm = __shfl_sync(kFullS, m, l);
      }
      run += __shfl_sync(kFullS, incl, 31);
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      peak = smax(peak, __shfl_xor_sync(kFullS, peak, off));
      busy += __shfl_xor_sync(kFullS, busy, off);
    }
    if (lane == 0) {
      s.peak[d] = peak;
      s.dest_bytes[d] = vt;
      s.dest_cnt[d] = vj;
      s.xfree[d] = vm;
      s.dev3n[3 * d + 1] = busy;
    }
  }
  __syncthreads();
  if (tid != 0) return;
  int vd = -1;
  for (int d = 0; d < n; ++d) {
    const int64_t t = s.dest_bytes[d];
    if (t == INT64_MAX) continue;
    if (vd < 0 || t < s.dest_bytes[vd] || (t == s.dest_bytes[vd] && s.dest_cnt[d] < s.dest_cnt[vd])) vd = d;
  }
  if (vd >= 0) {
    err->status = kInfeasible;
    err->code = E_SIM_MEMORY;
    err->a = vd;
    err->b = s.dest_bytes[vd];
    err->c = s.dest_cnt[vd];
    err->d = s.xfree[vd];
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
  const int64_t makespan = sh_mk;
  for (int d = 0; d < n; ++d) {
    s.dev3n[3 * d + 0] = s.peak[d];
    s.dev3n[3 * d + 2] = makespan - s.dev3n[3 * d + 1];
  }
  *s.makespan = makespan;
  s.xfer4[0] = static_cast<int64_t>(sh_x[0]);
  s.xfer4[1] = static_cast<int64_t>(sh_x[1]);
  s.xfer4[2] = 0;  // a tensor is sent once per device: duplicates never arise
  s.xfer4[3] = static_cast<int64_t>(sh_x[2] - sh_x[0]);
  err->status = kOk;
  err->code = E_NONE;
}

void launch_simulate(const DSim *sims, int nsims, const DGraph *graphs, cudaStream_t s) {
  constexpr int W = 4;
  k_simulate<W><<<(nsims + W - 1) / W, 32 * W, 0, s>>>(sims, nsims, graphs);
  // one CTA per problem; a lone problem gets the widest CTA for its edge passes
  k_sim_flow<<<nsims, nsims <= 148 ? 1024 : 256, 0, s>>>(sims, nsims, graphs);
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

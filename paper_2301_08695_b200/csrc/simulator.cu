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

void launch_simulate(const DSim *sims, int nsims, const DGraph *graphs, cudaStream_t s) {
  constexpr int W = 4;
  k_simulate<W><<<(nsims + W - 1) / W, 32 * W, 0, s>>>(sims, nsims, graphs);
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

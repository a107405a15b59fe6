// Scheduling helpers shared by the list placer (K2, listsched.cu) and the
// m-TOPO placer (placer.cu): the placer context, the schedulable-time fold
// (placers.cpp:43-101), warp reductions and the exec-order emission.
#pragma once
#include "bx_device.cuh"

namespace bx {

constexpr unsigned kFull = 0xffffffffu;
constexpr int64_t kInf = INT64_MAX;

// ---------------------------------------------------------------- K2 ----
struct Ctx {
  int V, n, mode, sct;
  // parallel comm on a graph whose every producer sends the same bytes on
  // all its out-edges: a cache arrival (finish + the same c) never changes a
  // term, so the cache is neither read nor written
  bool nocache = false;
  const int64_t *k, *need, *in_c, *cap;
  const int32_t *in_off, *in_src, *out_off, *out_dst, *fav;
  int64_t cmax;
  // ready slots (list placer): column-major key matrix Kc[q * V + slot],
  // dead flags deadc[q * V + slot], node / urgency / live-pair count per slot
  int64_t *Kc, *cache, *finish, *urg_s, *start;
  uint8_t *deadc;
  int32_t *pending, *alive_s, *node_s, *rpos, *device_of, *cseq, *nc;
  int64_t *scv;
  int32_t *scg;
  // per in-CSR slot x of a ready node: its parent's device and finish time,
  // written when the parent commits (inpos maps out-edge -> in-CSR slot)
  int32_t *pdev;
  int64_t *pfin;
  const int32_t *inpos;
  // shared memory, per warp
  int64_t *F, *tail, *res, *capS, *awu;
  int32_t *awf, *excl;
};

__device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// schedulable_time_impl (placers.cpp:43-79) as an estimate. Parallel mode
// returns the data-ready time (t0 = 0 gives the max over parent terms);
// sequential mode folds the queue tails in ascending in-edge order (the
// reference folds a copy of them; the running term stands in for the copy).
__device__ __forceinline__ int64_t est_time(const Ctx &c, int j, int p, int64_t t0, int32_t &gen) {
  int64_t t = t0;
  const int b = __ldg(c.in_off + (j)), e = __ldg(c.in_off + (j + 1));
  const int n = c.n;
  if (c.mode == 1) {
    for (int x = b; x < e; ++x) {
      int i = __ldg(c.in_src + (x));
      int q = c.device_of[i];
      int64_t fin = c.finish[i];
      int64_t term;
      if (q == p) {
        term = fin;
      } else {
        int64_t cached = c.cache[static_cast<int64_t>(i) * n + p];
        term = cached >= 0 ? max64(fin, cached) : fin + __ldg(c.in_c + (x));
      }
      t = max64(t, term);
    }
  } else {
    // no copy of the tails: after the first new transfer the copy's tail of
    // p is the running term T and every device touched since holds a value
    // <= T, so a transfer from q starts at max(finish, T, tail[q]) on the
    // LIVE tails
    (void)gen;
    int64_t T = c.tail[p];
    for (int x = b; x < e; ++x) {
      const int i = __ldg(c.in_src + (x));
      const int q = c.device_of[i];
      const int64_t fin = c.finish[i];
      const bool local = q == p;
      const int64_t cached = local ? -1 : c.cache[static_cast<int64_t>(i) * n + p];
      const bool xfer = !local && cached < 0;
      const int64_t tn = max64(max64(fin, T), c.tail[q]) + __ldg(c.in_c + (x));
      const int64_t term = local ? fin : (xfer ? tn : max64(fin, cached));
      T = xfer ? tn : T;
      t = max64(t, term);
    }
  }
  return t;
}

// Stored key component for (j, p): data-ready time (parallel) or the full
// schedulable time as a lower bound (sequential).
__device__ __forceinline__ int64_t row_value(const Ctx &c, int j, int p, int32_t &gen) {
  return c.mode == 1 ? est_time(c, j, p, 0, gen) : est_time(c, j, p, c.F[p], gen);
}

// commit_schedulable_time (placers.cpp:95-101): replays the fold on the live
// tails, records arrival times in the cache and lists the parents whose
// tensor just landed on p. Single lane.
static __device__ int64_t commit_fold(const Ctx &c, int j, int p, int *count) {
  int cnt = 0;
  const int n = c.n;
  int64_t t = c.F[p];
  for (int x = __ldg(c.in_off + (j)); x < __ldg(c.in_off + (j + 1)); ++x) {
    int i = __ldg(c.in_src + (x));
    int q = c.device_of[i];
    int64_t fin = c.finish[i];
    if (q == p) {
      t = max64(t, fin);
      continue;
    }
    int64_t *slot = c.cache + static_cast<int64_t>(i) * n + p;
    if (*slot >= 0) {
      t = max64(t, max64(fin, *slot));
      continue;
    }
    int64_t term;
    if (c.mode == 1) {
      term = fin + __ldg(c.in_c + (x));
    } else {
      term = max64(fin, max64(c.tail[q], c.tail[p])) + __ldg(c.in_c + (x));
      c.tail[q] = term;
      c.tail[p] = term;
    }
    *slot = term;
    c.nc[cnt++] = i;
    t = max64(t, term);
  }
  *count = cnt;
  return t;
}

__device__ __forceinline__ bool lex_less(int64_t t1, int64_t i1, int64_t t2, int64_t i2) {
  return t1 < t2 || (t1 == t2 && i1 < i2);
}

__device__ __forceinline__ void warp_argmin(int64_t &t, int64_t &idx) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    int64_t t2 = __shfl_xor_sync(kFull, t, o);
    int64_t i2 = __shfl_xor_sync(kFull, idx, o);
    if (lex_less(t2, i2, t, idx)) {
      t = t2;
      idx = i2;
    }
  }
}

// Lexicographic (key, id) warp argmin for non-negative int64 keys and 32-bit
// ids with three REDUX instructions instead of 20 shuffles: min of the key's
// high word, then of the low word among lanes holding that high word, then
// of the id among lanes holding the minimum key. Every lane gets the result.
__device__ __forceinline__ void warp_argmin_u(int64_t &t, unsigned &id) {
  const unsigned long long u = static_cast<unsigned long long>(t);
  const unsigned hi = static_cast<unsigned>(u >> 32), lo = static_cast<unsigned>(u);
  const unsigned mhi = __reduce_min_sync(kFull, hi);
  const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
  const bool win = hi == mhi && lo == mlo;
  id = __reduce_min_sync(kFull, win ? id : 0xffffffffu);
  t = static_cast<int64_t>((static_cast<unsigned long long>(mhi) << 32) | mlo);
}

__device__ __forceinline__ int64_t warp_max64(int64_t v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = max64(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ int warp_min_i32(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = min(v, __shfl_xor_sync(kFull, v, o));
  return v;
}

__device__ __forceinline__ void set_err(DErr *e, int status, int code, int64_t a, int64_t b) {
  e->status = status;
  e->code = code;
  e->a = a;
  e->b = b;
}

// exec_order (placers.cpp:282-294): nodes sorted by (start, index), appended
// per device. Commits on one device happen in non-decreasing start order,
// so a stable scatter of the commit sequence by device is already sorted by
// start; only runs of equal start (zero-duration nodes) need re-sorting by
// index.
static __device__ void emit_exec_order(const Ctx &c, const DJob &jb, int32_t *cntS, int lane) {
  const int V = c.V, n = c.n;
  for (int d = lane; d < n; d += 32) cntS[d] = 0;
  __syncwarp();
  for (int j = lane; j < V; j += 32) atomicAdd(&cntS[c.device_of[j]], 1);
  __syncwarp();
  if (lane == 0) {
    int acc = 0;
    for (int d = 0; d < n; ++d) {
      int v = cntS[d];
      jb.exec_off[d] = acc;
      cntS[d] = acc;
      acc += v;
    }
    jb.exec_off[n] = acc;
  }
  __syncwarp();
  const unsigned lt = (1u << lane) - 1u;
  for (int base = 0; base < V; base += 32) {
    int x = base + lane;
    bool act = x < V;
    unsigned am = __ballot_sync(kFull, act);
    if (act) {
      int j = c.cseq[x];
      int d = c.device_of[j];
      unsigned m = __match_any_sync(am, d);
      int rank = __popc(m & lt);
      jb.exec_order[cntS[d] + rank] = j;
      __syncwarp(am);
      if (rank == 0) cntS[d] += __popc(m);
    }
    __syncwarp();
  }
  __syncwarp();
  // equal-start runs must be ascending by index
  bool bad = false;
  for (int x = lane; x + 1 < V; x += 32) {
    int a = jb.exec_order[x], b = jb.exec_order[x + 1];
    if (c.device_of[a] == c.device_of[b] && c.start[a] == c.start[b] && a > b) bad = true;
  }
  if (__any_sync(kFull, bad) && lane == 0) {
    for (int d = 0; d < n; ++d) {
      int lo = jb.exec_off[d], hi = jb.exec_off[d + 1];
      for (int x = lo + 1; x < hi; ++x) {
        int v = jb.exec_order[x];
        int64_t s = c.start[v];
        int y = x - 1;
        while (y >= lo && c.start[jb.exec_order[y]] == s && jb.exec_order[y] > v) {
          jb.exec_order[y + 1] = jb.exec_order[y];
          --y;
        }
        jb.exec_order[y + 1] = v;
      }
    }
  }
  __syncwarp();
}

// Appends the nodes of `cand` (lane-local flag) to the ready list.
__device__ __forceinline__ int ready_append(const Ctx &c, int R, bool flag, int node, int lane) {
  unsigned m = __ballot_sync(kFull, flag);
  if (flag) {
    int pos = R + __popc(m & ((1u << lane) - 1u));
    c.node_s[pos] = node;
    c.rpos[node] = pos;
  }
  return R + __popc(m);
}

// m-SCT urgency (placers.cpp:259-266): latest parent finish plus the full
// transfer time, ignoring caches and queues.
__device__ __forceinline__ int64_t urgency(const Ctx &c, int j) {
  int64_t u = 0;
  for (int x = __ldg(c.in_off + (j)); x < __ldg(c.in_off + (j + 1)); ++x) u = max64(u, c.finish[__ldg(c.in_src + (x))] + __ldg(c.in_c + (x)));
  return u;
}


}  // namespace bx

// K1 (ingest) and K2 (list placer) for sm_100a.
//
// K2 restates place_list (proj/src/placers.cpp:115-295) in its exact-argmin
// form (SURVEY.md finding 1): at every step the lexicographic minimum of
// (key(j,p), j, p) over all live (ready, unplaced, not dead, not excluded)
// pairs is either committed or discarded for memory. The reference reaches
// the same sequence through a lazy min-heap with re-pushes (:188-202).
//
// One warp owns one placement problem for its whole life (a persistent
// scheduling loop: no per-step launches). Per-device state (dev_free, queue
// tails, reservations, awake reservations) lives in shared memory; per-node
// state and the key matrix live in HBM/L2. Keys are kept incrementally:
//   * parallel comm mode: K[j][p] = data-ready time of j on p (max over
//     parents of the arrival term, placers.cpp:55-61); key = max(dev_free[p],
//     K[j][p]) is formed during the scan, so a commit only has to touch the
//     rows of newly ready children and the entries of consumers whose parent
//     tensor just got cached on p;
//   * sequential comm mode: queue tails only grow, so a key computed earlier
//     is a lower bound of the current key; K[j][p] holds that lower bound and
//     the winner of a scan is re-keyed exactly (the lazy-heap argument of
//     placers.cpp:198-202) before it may commit.
// m-SCT's awake floor (placers.cpp:147-156) is applied during the scan from
// the live awake_for/awake_until/urgent values, so lifting a reservation
// needs no re-keying at all.
#include <cub/cub.cuh>

#include "bx_device.cuh"

namespace bx {

constexpr unsigned kFull = 0xffffffffu;
constexpr int64_t kInf = INT64_MAX;

// ---------------------------------------------------------------- K1 ----
// Per (graph, comm model): in-CSR gather of src + comm_time per slot, and
// c_max. Bytes per edge: 4 (in_edge) + 4 (esrc) + 8 (ebytes) read, 4 + 8
// written.
__global__ void k_prep_edges(DGraph g, DPrep pr, int write_src) {
  int64_t best = 0;
  int neg = 0;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.E; x += gridDim.x * blockDim.x) {
    int e = g.in_edge[x];
    int64_t b = g.ebytes[e];
    if (b < 0) {
      neg = 1;
      b = 0;
    }
    if (write_src) g.in_src[x] = g.esrc[e];
    int64_t c = comm_time_exact(pr.ic, pr.pb, b);
    pr.in_c[x] = c;
    best = c > best ? c : best;
  }
  // warp max then one atomic per warp
  for (int o = 16; o > 0; o >>= 1) {
    int64_t v = __shfl_xor_sync(kFull, best, o);
    best = v > best ? v : best;
    neg |= __shfl_xor_sync(kFull, neg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (best > 0) atomicMax(reinterpret_cast<unsigned long long *>(pr.cmax), static_cast<unsigned long long>(best));
    if (neg && write_src) atomicOr(&g.flags[1], 1);
  }
}

// need[j] = perm + out + temp (reserve_bytes, placers.hpp:43-45).
__global__ void k_prep_nodes(DGraph g) {
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < g.V; j += gridDim.x * blockDim.x) {
    int64_t v = g.perm[j] + g.outb[j] + g.temp[j];
    g.need[j] = v;
    g.iota[j] = j;
    g.indeg_left[j] = g.in_off[j + 1] - g.in_off[j];
  }
}

// Acyclicity (meta_topo_order's CycleError, transforms.cpp:446-479): the set
// of nodes Kahn's algorithm cannot peel does not depend on the pop order,
// so a level-synchronous peel finds the same residue. One CTA per graph;
// the frontier ping-pongs through `queue` (2*V ints of scratch).
__global__ void k_kahn(DGraph *graphs, int32_t *const *queues) {
  DGraph g = graphs[blockIdx.x];
  int32_t *q = queues[blockIdx.x];
  __shared__ int s_n[2];
  __shared__ int s_total;
  int V = g.V;
  if (threadIdx.x == 0) {
    s_n[0] = 0;
    s_n[1] = 0;
    s_total = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    if (g.indeg_left[j] == 0) q[atomicAdd(&s_n[0], 1)] = j;
  }
  __syncthreads();
  int cur = 0;
  while (true) {
    int cnt = s_n[cur];
    if (cnt == 0) break;
    int32_t *in = q + (cur ? V : 0);
    int32_t *out = q + (cur ? 0 : V);
    if (threadIdx.x == 0) s_total += cnt;
    for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
      int u = in[x];
      for (int y = g.out_off[u]; y < g.out_off[u + 1]; ++y) {
        int v = g.edst[y];
        if (atomicSub(&g.indeg_left[v], 1) == 1) out[atomicAdd(&s_n[cur ^ 1], 1)] = v;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) s_n[cur] = 0;
    cur ^= 1;
    __syncthreads();
  }
  if (threadIdx.x == 0) g.flags[0] = s_total;
}

// ---------------------------------------------------------------- K2 ----
struct Ctx {
  int V, n, mode, sct;
  const int64_t *k, *need, *in_c, *cap;
  const int32_t *in_off, *in_src, *out_off, *out_dst, *fav;
  int64_t cmax;
  int64_t *K, *cache, *finish, *urgent, *start;
  uint8_t *dead;
  int32_t *pending, *alive, *ready, *rpos, *device_of, *cseq, *nc;
  int64_t *scv;
  int32_t *scg;
  // shared memory, per warp
  int64_t *F, *tail, *res, *capS, *awu;
  int32_t *awf, *excl;
};

__device__ __forceinline__ int64_t max64(int64_t a, int64_t b) { return a > b ? a : b; }
__device__ __forceinline__ int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// schedulable_time_impl (placers.cpp:43-79) as an estimate. Parallel mode
// returns the data-ready time (t0 = 0 gives the max over parent terms);
// sequential mode folds the queue tails in ascending in-edge order through
// this lane's scratch copy (generation-tagged, so no copy is made).
__device__ __forceinline__ int64_t est_time(const Ctx &c, int j, int p, int64_t t0, int32_t &gen) {
  int64_t t = t0;
  const int b = c.in_off[j], e = c.in_off[j + 1];
  const int n = c.n;
  if (c.mode == 1) {
    for (int x = b; x < e; ++x) {
      int i = c.in_src[x];
      int q = c.device_of[i];
      int64_t fin = c.finish[i];
      int64_t term;
      if (q == p) {
        term = fin;
      } else {
        int64_t cached = c.cache[static_cast<int64_t>(i) * n + p];
        term = cached >= 0 ? max64(fin, cached) : fin + c.in_c[x];
      }
      t = max64(t, term);
    }
  } else {
    ++gen;
    for (int x = b; x < e; ++x) {
      int i = c.in_src[x];
      int q = c.device_of[i];
      int64_t fin = c.finish[i];
      int64_t term;
      if (q == p) {
        term = fin;
      } else {
        int64_t cached = c.cache[static_cast<int64_t>(i) * n + p];
        if (cached >= 0) {
          term = max64(fin, cached);
        } else {
          int64_t tq = c.scg[q] == gen ? c.scv[q] : c.tail[q];
          int64_t tp = c.scg[p] == gen ? c.scv[p] : c.tail[p];
          term = max64(fin, max64(tq, tp)) + c.in_c[x];
          c.scv[q] = term;
          c.scg[q] = gen;
          c.scv[p] = term;
          c.scg[p] = gen;
        }
      }
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
__device__ int64_t commit_fold(const Ctx &c, int j, int p, int *count) {
  int cnt = 0;
  const int n = c.n;
  int64_t t = c.F[p];
  for (int x = c.in_off[j]; x < c.in_off[j + 1]; ++x) {
    int i = c.in_src[x];
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
      term = fin + c.in_c[x];
    } else {
      term = max64(fin, max64(c.tail[q], c.tail[p])) + c.in_c[x];
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
__device__ void emit_exec_order(const Ctx &c, const DJob &jb, int32_t *cntS, int lane) {
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
    c.ready[pos] = node;
    c.rpos[node] = pos;
  }
  return R + __popc(m);
}

// m-SCT urgency (placers.cpp:259-266): latest parent finish plus the full
// transfer time, ignoring caches and queues.
__device__ __forceinline__ int64_t urgency(const Ctx &c, int j) {
  int64_t u = 0;
  for (int x = c.in_off[j]; x < c.in_off[j + 1]; ++x) u = max64(u, c.finish[c.in_src[x]] + c.in_c[x]);
  return u;
}

template <int kWarps>
__global__ void __launch_bounds__(32 * kWarps) k_place_list(const DJob *jobs, int njobs, const DGraph *graphs,
                                                           const DPrep *preps, int maxn) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jid = blockIdx.x * kWarps + warp;
  if (jid >= njobs) return;
  const DJob jb = jobs[jid];
  if (jb.skip || jb.algo == 0) return;
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  // acyclicity then byte-count validation, in the reference's order
  if (g.flags[0] != g.V) {
    if (lane == 0) set_err(jb.err, kValidation, E_CYCLE, 0, 0);
    return;
  }
  if (g.flags[1]) {
    if (lane == 0) set_err(jb.err, kValidation, E_NEG_BYTES, 0, 0);
    return;
  }

  Ctx c;
  c.V = g.V;
  c.n = jb.n;
  c.mode = jb.mode;
  c.sct = (jb.algo == 2 && jb.fav != nullptr);
  c.k = g.k;
  c.need = g.need;
  c.in_c = pr.in_c;
  c.cap = jb.cap;
  c.in_off = g.in_off;
  c.in_src = g.in_src;
  c.out_off = g.out_off;
  c.out_dst = g.edst;
  c.fav = jb.fav;
  c.cmax = *pr.cmax;
  c.K = jb.K;
  c.cache = jb.cache;
  c.finish = jb.finish;
  c.urgent = jb.urgent;
  c.start = jb.start;
  c.dead = jb.dead;
  c.pending = jb.pending;
  c.alive = jb.alive;
  c.ready = jb.ready;
  c.rpos = jb.rpos;
  c.device_of = jb.device_of;
  c.cseq = jb.cseq;
  c.nc = jb.nc;
  c.scv = jb.sc_val + static_cast<int64_t>(lane) * jb.n;
  c.scg = jb.sc_gen + static_cast<int64_t>(lane) * jb.n;
  {
    unsigned char *base = smem + static_cast<size_t>(warp) * (maxn * 56);
    c.F = reinterpret_cast<int64_t *>(base);
    c.tail = c.F + maxn;
    c.res = c.tail + maxn;
    c.capS = c.res + maxn;
    c.awu = c.capS + maxn;
    c.awf = reinterpret_cast<int32_t *>(c.awu + maxn);
    c.excl = c.awf + maxn;
  }
  const int V = c.V, n = c.n;
  for (int d = lane; d < n; d += 32) {
    c.F[d] = 0;
    c.tail[d] = 0;
    c.res[d] = 0;
    c.capS[d] = c.cap[d];
    c.awu[d] = 0;
    c.awf[d] = -1;
    c.excl[d] = 0;
  }
  // per-node init + initial ready set (sources), keys 0 (dev_free = 0)
  int R = 0;
  for (int base = 0; base < V; base += 32) {
    int j = base + lane;
    bool src = false;
    if (j < V) {
      int indeg = g.in_off[j + 1] - g.in_off[j];
      c.pending[j] = indeg;
      c.alive[j] = n;
      c.device_of[j] = -1;
      c.finish[j] = 0;
      c.urgent[j] = 0;
      src = indeg == 0;
    }
    R = ready_append(c, R, src, j, lane);
  }
  __syncwarp();
  for (int r = lane; r < R * n; r += 32) c.K[static_cast<int64_t>(c.ready[r / n]) * n + (r % n)] = 0;
  __syncwarp();

  int32_t gen = 0;
  int placed = 0;
  int64_t discarded = 0, excluded = 0, awake = 0;
  int minptr = 0;  // lane 0: first possibly-unplaced slot of need_order

  while (placed < V) {
    // ---- scan: exact key of every live pair, lexicographic argmin --------
    int64_t bt = kInf, bi = kInf;
    const int total = R * n;
    for (int r = lane; r < total; r += 32) {
      int s = r / n;
      int p = r - s * n;
      int j = c.ready[s];
      int64_t cell = static_cast<int64_t>(j) * n + p;
      if (c.excl[p] || c.dead[cell]) continue;
      int64_t t = max64(c.K[cell], c.F[p]);
      if (c.sct) {
        int aw = c.awf[p];
        if (aw >= 0 && aw != j) t = max64(t, min64(c.awu[p], c.urgent[j]));
      }
      if (lex_less(t, cell, bt, bi)) {
        bt = t;
        bi = cell;
      }
    }
    warp_argmin(bt, bi);
    if (bi == kInf) {
      if (lane == 0) set_err(jb.err, kInfeasible, E_NO_PAIR, 0, 0);
      return;
    }
    const int j = static_cast<int>(bi / n);
    const int p = static_cast<int>(bi - static_cast<int64_t>(j) * n);
    const int64_t t = bt;

    if (c.mode == 0) {
      // lazy re-key of the winner (placers.cpp:198-202)
      int64_t fresh = 0;
      if (lane == 0) fresh = est_time(c, j, p, c.F[p], gen);
      fresh = __shfl_sync(kFull, fresh, 0);
      int64_t key = fresh;
      if (c.sct) {
        int aw = c.awf[p];
        if (aw >= 0 && aw != j) key = max64(key, min64(c.awu[p], c.urgent[j]));
      }
      if (key != t) {
        if (lane == 0) c.K[bi] = fresh;
        __syncwarp();
        continue;
      }
    }

    const int64_t needj = c.need[j];
    if (c.res[p] + needj > c.capS[p]) {
      // discard (placers.cpp:203-219)
      int left = 0;
      if (lane == 0) {
        c.dead[bi] = 1;
        left = --c.alive[j];
      }
      left = __shfl_sync(kFull, left, 0);
      if (left == 0) {
        if (lane == 0) set_err(jb.err, kInfeasible, E_FITS_NONE, j, 0);
        return;
      }
      ++discarded;
      // smallest need among all unplaced nodes (the `remaining` multiset,
      // placers.cpp:126,208): first unplaced node in ascending-need order
      int64_t minrem = 0;
      if (lane == 0) {
        while (c.device_of[g.need_order[minptr]] >= 0) ++minptr;
        minrem = c.need[g.need_order[minptr]];
      }
      minrem = __shfl_sync(kFull, minrem, 0);
      if (c.res[p] + minrem > c.capS[p]) {
        ++excluded;
        int first_dead = INT32_MAX;
        for (int j2 = lane; j2 < V; j2 += 32) {
          if (c.device_of[j2] < 0) {
            int64_t cell = static_cast<int64_t>(j2) * n + p;
            if (!c.dead[cell]) {
              c.dead[cell] = 1;
              if (--c.alive[j2] == 0) first_dead = min(first_dead, j2);
            }
          }
        }
        first_dead = warp_min_i32(first_dead);
        if (first_dead != INT32_MAX) {
          if (lane == 0) set_err(jb.err, kInfeasible, E_FITS_NONE, first_dead, 0);
          return;
        }
        if (lane == 0) c.excl[p] = 1;
      }
      __syncwarp();
      continue;
    }

    // ---- commit (placers.cpp:221-233) ------------------------------------
    const int64_t fin = t + c.k[j];
    int ncount = 0;
    if (lane == 0) {
      c.device_of[j] = p;
      c.start[j] = t;
      c.finish[j] = fin;
      commit_fold(c, j, p, &ncount);
      c.F[p] = fin;
      c.res[p] += needj;
      c.cseq[placed] = j;
      // swap-remove j from the ready list
      int pos = c.rpos[j];
      int last = c.ready[R - 1];
      c.ready[pos] = last;
      c.rpos[last] = pos;
    }
    ncount = __shfl_sync(kFull, ncount, 0);
    ++placed;
    --R;
    if (c.sct) {
      // awake reservations (placers.cpp:235-254)
      int got = 0;
      if (lane == 0) {
        c.awf[p] = -1;
        for (int q = 0; q < n; ++q)
          if (c.awf[q] == j) c.awf[q] = -1;
        int h = c.fav[j];
        if (h >= 0 && c.device_of[h] < 0) {
          c.awf[p] = h;
          c.awu[p] = fin + c.cmax;
          got = 1;
        }
      }
      awake += __shfl_sync(kFull, got, 0);
    }
    __syncwarp();

    // ---- readiness (placers.cpp:256-268) ---------------------------------
    const int R0 = R;
    for (int base = c.out_off[j]; base < c.out_off[j + 1]; base += 32) {
      int y = base + lane;
      bool fresh = false;
      int child = -1;
      if (y < c.out_off[j + 1]) {
        child = c.out_dst[y];
        fresh = --c.pending[child] == 0;
      }
      R = ready_append(c, R, fresh, child, lane);
    }
    __syncwarp();
    const int nnew = R - R0;
    if (nnew > 0) {
      if (c.sct) {
        for (int s = lane; s < nnew; s += 32) {
          int ch = c.ready[R0 + s];
          c.urgent[ch] = urgency(c, ch);
        }
      }
      for (int r = lane; r < nnew * n; r += 32) {
        int s = r / n;
        int q = r - s * n;
        int ch = c.ready[R0 + s];
        c.K[static_cast<int64_t>(ch) * n + q] = row_value(c, ch, q, gen);
      }
    }
    // ---- cached parents lower their other consumers' keys on p (:271-279)
    for (int a = 0; a < ncount; ++a) {
      int i = c.nc[a];
      for (int y = c.out_off[i] + lane; y < c.out_off[i + 1]; y += 32) {
        int cc = c.out_dst[y];
        if (cc == j || c.device_of[cc] >= 0 || c.pending[cc] != 0) continue;
        int64_t cell = static_cast<int64_t>(cc) * n + p;
        if (c.dead[cell]) continue;
        c.K[cell] = row_value(c, cc, p, gen);
      }
    }
    __syncwarp();
  }

  // sorted exec lists
  emit_exec_order(c, jb, reinterpret_cast<int32_t *>(c.excl) , lane);
  if (lane == 0) {
    jb.stats[0] = discarded;
    jb.stats[1] = excluded;
    jb.stats[2] = awake;
    set_err(jb.err, kOk, E_NONE, 0, 0);
  }
}

// ------------------------------------------------------------ m-TOPO ----
// place_mtopo (placers.cpp:314-365): min-index Kahn order, balanced fill,
// then the schedule estimate with commit_schedulable_time. One warp per job.
template <int kWarps>
__global__ void __launch_bounds__(32 * kWarps) k_place_topo(const DJob *jobs, int njobs, const DGraph *graphs,
                                                           const DPrep *preps, int maxn) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int jid = blockIdx.x * kWarps + warp;
  if (jid >= njobs) return;
  const DJob jb = jobs[jid];
  if (jb.skip || jb.algo != 0) return;
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  const int V = g.V, n = jb.n;
  // cap = ceil(total / n) + largest; infeasible before the acyclicity check
  int64_t total = 0, largest = 0;
  for (int j = lane; j < V; j += 32) {
    int64_t b = g.need[j];
    total += b;
    largest = max64(largest, b);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) total += __shfl_xor_sync(kFull, total, o);
  largest = warp_max64(largest);
  int64_t mincap = jb.cap[0];
  for (int d = 1; d < n; ++d) mincap = min64(mincap, jb.cap[d]);
  const int64_t cap = (total + n - 1) / n + largest;
  if (cap > mincap) {
    if (lane == 0) set_err(jb.err, kInfeasible, E_TOPO_CAP, cap, mincap);
    return;
  }
  if (g.flags[0] != V) {
    if (lane == 0) set_err(jb.err, kValidation, E_CYCLE, 0, 0);
    return;
  }

  Ctx c;
  c.V = V;
  c.n = n;
  c.mode = jb.mode;
  c.in_c = pr.in_c;
  c.in_off = g.in_off;
  c.in_src = g.in_src;
  c.cache = jb.cache;
  c.finish = jb.finish;
  c.device_of = jb.device_of;
  c.nc = jb.nc;
  {
    unsigned char *base = smem + static_cast<size_t>(warp) * (maxn * 56);
    c.F = reinterpret_cast<int64_t *>(base);
    c.tail = c.F + maxn;
  }
  for (int d = lane; d < n; d += 32) {
    c.F[d] = 0;
    c.tail[d] = 0;
  }
  int32_t *order = jb.exec_order;  // topo order doubles as the exec lists
  int R = 0;
  for (int base = 0; base < V; base += 32) {
    int j = base + lane;
    bool src = false;
    if (j < V) {
      int indeg = g.in_off[j + 1] - g.in_off[j];
      jb.pending[j] = indeg;
      jb.device_of[j] = -1;
      jb.finish[j] = 0;
      src = indeg == 0;
    }
    unsigned m = __ballot_sync(kFull, src);
    if (src) jb.ready[R + __popc(m & ((1u << lane) - 1u))] = j;
    R += __popc(m);
  }
  __syncwarp();
  // min-index Kahn (transforms.cpp:446-479)
  for (int cnt = 0; cnt < V; ++cnt) {
    int best = INT32_MAX, bpos = -1;
    for (int s = lane; s < R; s += 32) {
      int v = jb.ready[s];
      if (v < best) {
        best = v;
        bpos = s;
      }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      int b2 = __shfl_xor_sync(kFull, best, o);
      int p2 = __shfl_xor_sync(kFull, bpos, o);
      if (b2 < best) {
        best = b2;
        bpos = p2;
      }
    }
    if (lane == 0) {
      order[cnt] = best;
      jb.ready[bpos] = jb.ready[R - 1];
    }
    --R;
    __syncwarp();
    for (int base = g.out_off[best]; base < g.out_off[best + 1]; base += 32) {
      int y = base + lane;
      bool fresh = false;
      int child = -1;
      if (y < g.out_off[best + 1]) {
        child = g.edst[y];
        fresh = --jb.pending[child] == 0;
      }
      unsigned m = __ballot_sync(kFull, fresh);
      if (fresh) jb.ready[R + __popc(m & ((1u << lane) - 1u))] = child;
      R += __popc(m);
    }
    __syncwarp();
  }
  if (lane == 0) {
    // balanced fill; the last device absorbs the rest (placers.cpp:337-347)
    int dev = 0;
    int64_t used = 0;
    jb.exec_off[0] = 0;
    for (int x = 0; x < V; ++x) {
      int j = order[x];
      int64_t b = g.need[j];
      if (used + b > cap && dev + 1 < n) {
        jb.exec_off[dev + 1] = x;
        ++dev;
        used = 0;
      }
      jb.device_of[j] = dev;
      used += b;
    }
    for (int d = dev + 1; d <= n; ++d) jb.exec_off[d] = V;
    // schedule estimate (placers.cpp:350-362); placement is fixed up front,
    // so every device_of is set before the fold runs
    for (int x = 0; x < V; ++x) {
      int j = order[x];
      int p = jb.device_of[j];
      // the reference writes st.device_of[j] lazily; parents precede j in
      // topo order, so the fold only reads already-visited nodes
      int cnt;
      int64_t t = commit_fold(c, j, p, &cnt);
      jb.start[j] = t;
      jb.finish[j] = t + g.k[j];
      c.F[p] = jb.finish[j];
    }
    jb.stats[0] = jb.stats[1] = jb.stats[2] = 0;
    set_err(jb.err, kOk, E_NONE, 0, 0);
  }
}

// ------------------------------------------------------------ launch ----
template <int W>
static void launch_place(const DJob *jobs, int njobs, const DGraph *graphs, const DPrep *preps, int maxn, bool topo,
                         cudaStream_t s) {
  int blocks = (njobs + W - 1) / W;
  size_t sm = static_cast<size_t>(W) * maxn * 56;
  if (topo) {
    k_place_topo<W><<<blocks, 32 * W, sm, s>>>(jobs, njobs, graphs, preps, maxn);
  } else {
    k_place_list<W><<<blocks, 32 * W, sm, s>>>(jobs, njobs, graphs, preps, maxn);
  }
}

void launch_prep(const DGraph &g, const DPrep &pr, bool first, cudaStream_t s) {
  if (first) {
    int nb = (g.V + 255) / 256;
    if (nb > 0) k_prep_nodes<<<nb < 1184 ? nb : 1184, 256, 0, s>>>(g);
  }
  int eb = (g.E + 255) / 256;
  if (eb > 0) k_prep_edges<<<eb < 1184 ? eb : 1184, 256, 0, s>>>(g, pr, first ? 1 : 0);
}

void launch_kahn(DGraph *graphs_dev, int32_t *const *queues_dev, int ngraphs, cudaStream_t s) {
  k_kahn<<<ngraphs, 512, 0, s>>>(graphs_dev, queues_dev);
}

// need_order: node indices by ascending (need, index); the radix sort is
// stable, so equal needs keep ascending index order.
cudaError_t sort_needs(void *tmp, size_t &tmp_bytes, const DGraph &g, int end_bit, cudaStream_t s) {
  return cub::DeviceRadixSort::SortPairs(tmp, tmp_bytes, g.need, g.need_keys, g.iota, g.need_order, g.V, 0, end_bit,
                                         s);
}

void launch_placers(const DJob *jobs, int njobs, const DGraph *graphs, const DPrep *preps, int maxn, bool any_topo,
                    bool any_list, cudaStream_t s) {
  // one warp per job; 4 jobs per CTA keeps many CTAs resident per SM for
  // batched sweeps while single-job launches stay one warp.
  if (any_list) launch_place<4>(jobs, njobs, graphs, preps, maxn, false, s);
  if (any_topo) launch_place<4>(jobs, njobs, graphs, preps, maxn, true, s);
}

}  // namespace bx

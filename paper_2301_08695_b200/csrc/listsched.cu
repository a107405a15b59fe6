// K2 — the m-ETF / m-SCT list placer for sm_100a.
//
// Restates place_list (proj/src/placers.cpp:115-295) in its exact-argmin
// form (SURVEY.md finding 1): at every step the lexicographic minimum of
// (key(j,p), j, p) over all live (ready, unplaced, not dead, not excluded)
// pairs is either committed or discarded for memory. The reference reaches
// the same sequence through a lazy min-heap with re-pushes (:188-202).
//
// One warp owns one placement problem for its whole life: a persistent
// scheduling loop, no per-step launches. Layout:
//   * shared memory (per warp): per-device state — dev_free F, queue tails,
//     reservations, capacities, awake reservations, exclusion flags — and,
//     per device column q, the exact top-KT pairs of that column as a sorted
//     list of (key, node) plus dirty/complete flags;
//   * HBM/L2: ready slots. Kc[q*V + s] holds the key component of the node in
//     slot s on device q, column-major so a column rescan is one coalesced
//     256-byte load per warp instruction; deadc[q*V + s] marks discarded pairs.
// Key maintenance:
//   * parallel comm mode: Kc = data-ready time (max over parents of the
//     arrival term, placers.cpp:55-61); key = max(F[q], Kc, m-SCT floor) is
//     formed when a column is scanned;
//   * sequential comm mode: queue tails only grow, so a key computed earlier
//     is a lower bound; the step's winner is re-keyed exactly before it may
//     commit (the lazy-heap argument of placers.cpp:198-202).
// A commit on device p changes column p (F[p], cached parents) and nothing
// else except removing the committed node from every column; so per step
// only column p is rescanned, every other column just drops the node from
// its top list, and new ready rows are merged into the lists. A column is
// rescanned only when its list runs dry or its keys change (m-SCT awake
// reservations, sequential re-keys).
#include "sched_common.cuh"

namespace bx {

constexpr int KT = 4;  // exact top-KT pairs kept per device column

struct Tops {
  int64_t *t;    // [n*KT] keys, ascending
  int32_t *j;    // [n*KT] nodes
  int32_t *cnt;  // [n]
  int32_t *flg;  // [n] bit0 dirty, bit1 complete (list holds every live pair)
};
constexpr int kDirty = 1, kComplete = 2;

__device__ __forceinline__ int64_t col_key(const Ctx &c, int q, int s, int j) {
  int64_t t = max64(c.Kc[static_cast<int64_t>(q) * c.V + s], c.F[q]);
  if (c.sct) {
    int aw = c.awf[q];
    if (aw >= 0 && aw != j) t = max64(t, min64(c.awu[q], c.urg_s[s]));
  }
  return t;
}

// Warp rescan of column q over ready slots [0, R): exact top-KT list.
__device__ void rescan(const Ctx &c, const Tops &T, int q, int R, int lane) {
  int64_t lt[KT];
  int lj[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    lt[k] = kInf;
    lj[k] = INT32_MAX;
  }
  int live = 0;
  const uint8_t *dcol = c.deadc + static_cast<int64_t>(q) * c.V;
  for (int s = lane; s < R; s += 32) {
    if (dcol[s]) continue;
    ++live;
    int j = c.node_s[s];
    int64_t t = col_key(c, q, s, j);
    if (lex_less(t, j, lt[KT - 1], lj[KT - 1])) {
      lt[KT - 1] = t;
      lj[KT - 1] = j;
#pragma unroll
      for (int k = KT - 1; k > 0; --k) {
        if (lex_less(lt[k], lj[k], lt[k - 1], lj[k - 1])) {
          int64_t a = lt[k];
          lt[k] = lt[k - 1];
          lt[k - 1] = a;
          int b = lj[k];
          lj[k] = lj[k - 1];
          lj[k - 1] = b;
        }
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(kFull, live, o);
  int cnt = 0;
#pragma unroll
  for (int r = 0; r < KT; ++r) {
    int64_t bt = lt[0];
    int64_t bj = lj[0];
    warp_argmin(bt, bj);
    if (bt == kInf) break;
    if (lane == 0) {
      T.t[q * KT + r] = bt;
      T.j[q * KT + r] = static_cast<int>(bj);
    }
    ++cnt;
    if (lj[0] == bj) {  // the owning lane pops its head
#pragma unroll
      for (int k = 0; k < KT - 1; ++k) {
        lt[k] = lt[k + 1];
        lj[k] = lj[k + 1];
      }
      lt[KT - 1] = kInf;
      lj[KT - 1] = INT32_MAX;
    }
  }
  if (lane == 0) {
    T.cnt[q] = cnt;
    T.flg[q] = live <= KT ? kComplete : 0;
  }
}

// Lane-owned list edits (the lane with q % 32 == lane owns column q).
__device__ __forceinline__ void list_remove(const Tops &T, int q, int j) {
  int c = T.cnt[q];
  int at = -1;
  for (int k = 0; k < c; ++k)
    if (T.j[q * KT + k] == j) at = k;
  if (at < 0) return;
  for (int k = at; k + 1 < c; ++k) {
    T.t[q * KT + k] = T.t[q * KT + k + 1];
    T.j[q * KT + k] = T.j[q * KT + k + 1];
  }
  T.cnt[q] = --c;
  if (c == 0 && !(T.flg[q] & kComplete)) T.flg[q] |= kDirty;
}

__device__ __forceinline__ void list_insert(const Tops &T, int q, int64_t t, int j) {
  int c = T.cnt[q];
  int f = T.flg[q];
  if (f & kDirty) return;
  if (c == KT) {
    if (!lex_less(t, j, T.t[q * KT + KT - 1], T.j[q * KT + KT - 1])) {
      T.flg[q] = f & ~kComplete;  // a live pair now sits outside the list
      return;
    }
    T.flg[q] = f & ~kComplete;  // the dropped tail is no longer listed
    --c;
  } else if (!(f & kComplete)) {
    // incomplete list: only pairs that beat the last listed one are known
    if (c == 0 || !lex_less(t, j, T.t[q * KT + c - 1], T.j[q * KT + c - 1])) return;
  }
  int k = c;
  while (k > 0 && lex_less(t, j, T.t[q * KT + k - 1], T.j[q * KT + k - 1])) {
    T.t[q * KT + k] = T.t[q * KT + k - 1];
    T.j[q * KT + k] = T.j[q * KT + k - 1];
    --k;
  }
  T.t[q * KT + k] = t;
  T.j[q * KT + k] = j;
  T.cnt[q] = c + 1;
}

constexpr int kListSmemPerDevice = 5 * 8 + 2 * 4 + KT * 12 + 2 * 4;  // bytes per device column

// Latency breakdown (kProf builds only): cycles since the last mark are
// charged to a phase slot; lane 0's totals are written at the end.
#define BX_MARK(slot)                       \
  do {                                      \
    if (kProf) {                            \
      int64_t now_ = clock64();             \
      prof[slot] += now_ - prof_last;       \
      prof_last = now_;                     \
    }                                       \
  } while (0)

template <int kWarps, bool kProf>
__global__ void __launch_bounds__(32 * kWarps, 7) k_place_list(const DJob *jobs, const int32_t *order,
                                                                        int njobs, const DGraph *graphs,
                                                                        const DPrep *preps, int maxn) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t prof[kProfSlots];
  int64_t prof_last = 0;
  if (kProf) {
#pragma unroll
    for (int k = 0; k < kProfSlots; ++k) prof[k] = 0;
    prof_last = clock64();
  }
  const int64_t prof_t0 = kProf ? clock64() : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int slot_id = blockIdx.x * kWarps + warp;
  if (slot_id >= njobs) return;
  const DJob jb = jobs[order[slot_id]];
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
  c.Kc = jb.K;
  c.cache = jb.cache;
  c.finish = jb.finish;
  c.urg_s = jb.urgent;
  c.start = jb.start;
  c.deadc = jb.dead;
  c.pending = jb.pending;
  c.alive_s = jb.alive;
  c.node_s = jb.ready;
  c.rpos = jb.rpos;
  c.device_of = jb.device_of;
  c.cseq = jb.cseq;
  c.nc = jb.nc;
  c.scv = jb.sc_val + static_cast<int64_t>(lane) * jb.n;
  c.scg = jb.sc_gen + static_cast<int64_t>(lane) * jb.n;
  Tops T;
  {
    unsigned char *base = smem + static_cast<size_t>(warp) * (maxn * kListSmemPerDevice);
    c.F = reinterpret_cast<int64_t *>(base);
    c.tail = c.F + maxn;
    c.res = c.tail + maxn;
    c.capS = c.res + maxn;
    c.awu = c.capS + maxn;
    T.t = c.awu + maxn;
    c.awf = reinterpret_cast<int32_t *>(T.t + maxn * KT);
    c.excl = c.awf + maxn;
    T.j = c.excl + maxn;
    T.cnt = T.j + maxn * KT;
    T.flg = T.cnt + maxn;
  }
  const int V = c.V, n = c.n;
  const int64_t Vs = V;
  for (int d = lane; d < n; d += 32) {
    c.F[d] = 0;
    c.tail[d] = 0;
    c.res[d] = 0;
    c.capS[d] = c.cap[d];
    c.awu[d] = 0;
    c.awf[d] = -1;
    c.excl[d] = 0;
    T.cnt[d] = 0;
    T.flg[d] = kDirty;
  }
  // per-node init + initial ready slots (sources), keys 0 (dev_free = 0)
  int R = 0;
  for (int base = 0; base < V; base += 32) {
    int j = base + lane;
    bool src = false;
    if (j < V) {
      int indeg = g.in_off[j + 1] - g.in_off[j];
      c.pending[j] = indeg;
      c.device_of[j] = -1;
      c.finish[j] = 0;
      src = indeg == 0;
    }
    R = ready_append(c, R, src, j, lane);
  }
  __syncwarp();
  for (int s = lane; s < R; s += 32) {
    c.urg_s[s] = 0;
    c.alive_s[s] = n;
  }
  for (int q = 0; q < n; ++q)
    for (int s = lane; s < R; s += 32) {
      c.Kc[q * Vs + s] = 0;
      c.deadc[q * Vs + s] = 0;
    }
  __syncwarp();

  int32_t gen = 0;
  int placed = 0, nexcl = 0;
  int64_t discarded = 0, excluded = 0, awake = 0;
  int minptr = 0;  // lane 0: first possibly-unplaced slot of need_order

  if (kProf) prof_last = clock64();
  while (placed < V) {
    if (kProf) ++prof[P_STEPS];
    // ---- refresh dirty columns ------------------------------------------
    for (int q0 = 0; q0 < n; q0 += 32) {
      int q = q0 + lane;
      unsigned m = __ballot_sync(kFull, q < n && (T.flg[q] & kDirty) && !c.excl[q]);
      while (m) {
        int qq = q0 + __ffs(m) - 1;
        m &= m - 1;
        rescan(c, T, qq, R, lane);
        if (kProf) ++prof[P_RESCANS];
      }
    }
    __syncwarp();
    BX_MARK(P_RESCAN);
    // ---- argmin over column heads: lexicographic (key, node, device) ------
    int64_t bt = kInf, bi = kInf;
    for (int q = lane; q < n; q += 32) {
      if (c.excl[q] || T.cnt[q] == 0) continue;
      int64_t t = T.t[q * KT];
      int64_t cell = static_cast<int64_t>(T.j[q * KT]) * n + q;
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
    const int sj = c.rpos[j];
    BX_MARK(P_ARGMIN);

    if (c.mode == 0) {
      // lazy re-key of the winner (placers.cpp:198-202)
      int64_t fresh = 0;
      if (lane == 0) fresh = est_time(c, j, p, c.F[p], gen);
      fresh = __shfl_sync(kFull, fresh, 0);
      int64_t key = fresh;
      if (c.sct) {
        int aw = c.awf[p];
        if (aw >= 0 && aw != j) key = max64(key, min64(c.awu[p], c.urg_s[sj]));
      }
      if (key != t) {
        if (lane == 0) {
          c.Kc[p * Vs + sj] = fresh;
          T.flg[p] |= kDirty;
        }
        __syncwarp();
        BX_MARK(P_REKEY);
        continue;
      }
      BX_MARK(P_REKEY);
    }

    const int64_t needj = c.need[j];
    if (c.res[p] + needj > c.capS[p]) {
      // discard (placers.cpp:203-219)
      int left = 0;
      if (lane == 0) {
        c.deadc[p * Vs + sj] = 1;
        left = --c.alive_s[sj];
      }
      left = __shfl_sync(kFull, left, 0);
      if (left == 0) {
        if (lane == 0) set_err(jb.err, kInfeasible, E_FITS_NONE, j, 0);
        return;
      }
      ++discarded;
      if (lane == (p & 31)) list_remove(T, p, j);
      // smallest need among all unplaced nodes (the `remaining` multiset,
      // placers.cpp:126,208): first unplaced node in ascending-need order
      int64_t minrem = 0;
      if (lane == 0) {
        while (c.device_of[g.need_order[minptr]] >= 0) ++minptr;
        minrem = c.need[g.need_order[minptr]];
      }
      minrem = __shfl_sync(kFull, minrem, 0);
      if (c.res[p] + minrem > c.capS[p]) {
        // exclusion: every unplaced (j2, p) dies, ascending j2. Unready nodes
        // carry no discards, so they die together exactly when the last
        // device goes; ready ones are counted per slot.
        ++excluded;
        ++nexcl;
        int first_dead = INT32_MAX;
        for (int s = lane; s < R; s += 32) {
          if (!c.deadc[p * Vs + s]) {
            c.deadc[p * Vs + s] = 1;
            if (--c.alive_s[s] == 0) first_dead = min(first_dead, c.node_s[s]);
          }
        }
        if (nexcl == n) {
          for (int x = lane; x < V; x += 32)
            if (c.device_of[x] < 0) first_dead = min(first_dead, x);
        }
        first_dead = warp_min_i32(first_dead);
        if (first_dead != INT32_MAX) {
          if (lane == 0) set_err(jb.err, kInfeasible, E_FITS_NONE, first_dead, 0);
          return;
        }
        if (lane == 0) c.excl[p] = 1;
      }
      __syncwarp();
      BX_MARK(P_DISCARD);
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
    }
    ncount = __shfl_sync(kFull, ncount, 0);
    ++placed;
    if (kProf) ++prof[P_COMMITS];
    BX_MARK(P_COMMIT);
    // swap-remove slot sj: the last slot moves in
    const int last = R - 1;
    if (sj != last) {
      for (int q = lane; q < n; q += 32) {
        c.Kc[q * Vs + sj] = c.Kc[q * Vs + last];
        c.deadc[q * Vs + sj] = c.deadc[q * Vs + last];
      }
      if (lane == 0) {
        int mv = c.node_s[last];
        c.node_s[sj] = mv;
        c.urg_s[sj] = c.urg_s[last];
        c.alive_s[sj] = c.alive_s[last];
        c.rpos[mv] = sj;
      }
    }
    --R;
    // j leaves every column; column p's keys moved with F[p]
    for (int q = lane; q < n; q += 32) {
      if (q == p) T.flg[q] |= kDirty;
      else list_remove(T, q, j);
    }
    __syncwarp();  // list edits above are lane-owned; lane 0 edits flags below
    if (c.sct) {
      // awake reservations (placers.cpp:235-254); the floor is read live,
      // so a changed reservation only dirties its column
      int got = 0;
      if (lane == 0) {
        c.awf[p] = -1;
        for (int q = 0; q < n; ++q)
          if (c.awf[q] == j) {
            c.awf[q] = -1;
            T.flg[q] |= kDirty;
          }
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
    BX_MARK(P_REMOVE);

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
    BX_MARK(P_READY);
    const int nnew = R - R0;
    if (nnew > 0) {
      for (int s = R0 + lane; s < R; s += 32) {
        c.alive_s[s] = n - nexcl;
        c.urg_s[s] = c.sct ? urgency(c, c.node_s[s]) : 0;
      }
      for (int r = lane; r < nnew * n; r += 32) {
        int s = R0 + r / n;
        int q = r % n;
        c.Kc[q * Vs + s] = row_value(c, c.node_s[s], q, gen);
        c.deadc[q * Vs + s] = static_cast<uint8_t>(c.excl[q] != 0);
      }
    }
    __syncwarp();
    BX_MARK(P_ROWS);
    // ---- cached parents change their other consumers' keys on p (:271-279)
    for (int a = 0; a < ncount; ++a) {
      int i = c.nc[a];
      for (int y = c.out_off[i] + lane; y < c.out_off[i + 1]; y += 32) {
        int cc = c.out_dst[y];
        if (cc == j || c.device_of[cc] >= 0 || c.pending[cc] != 0) continue;
        int s = c.rpos[cc];
        if (s >= R0) continue;  // new rows were keyed after the cache update
        if (c.deadc[p * Vs + s]) continue;
        c.Kc[p * Vs + s] = row_value(c, cc, p, gen);
      }
    }
    __syncwarp();
    BX_MARK(P_CACHE);
    // ---- merge new rows into the clean column lists ------------------------
    if (nnew > 0) {
      for (int q = lane; q < n; q += 32) {
        if (c.excl[q] || (T.flg[q] & kDirty)) continue;
        for (int s = R0; s < R; ++s) {
          int node = c.node_s[s];
          list_insert(T, q, col_key(c, q, s, node), node);
        }
      }
    }
    __syncwarp();
    BX_MARK(P_INSERT);
  }

  emit_exec_order(c, jb, c.excl, lane);
  BX_MARK(P_EMIT);
  if (lane == 0) {
    jb.stats[0] = discarded;
    jb.stats[1] = excluded;
    jb.stats[2] = awake;
    set_err(jb.err, kOk, E_NONE, 0, 0);
    if (kProf && jb.prof) {
      prof[P_TOTAL] = clock64() - prof_t0;
      for (int k = 0; k < kProfSlots; ++k) jb.prof[k] = prof[k];
    }
  }
}

void launch_list(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                 int maxn, bool prof, cudaStream_t s) {
  constexpr int W = 4;
  int blocks = (njobs + W - 1) / W;
  size_t sm = static_cast<size_t>(W) * maxn * kListSmemPerDevice;
  if (prof) {
    if (sm > 48 * 1024)
      cudaFuncSetAttribute(k_place_list<W, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    k_place_list<W, true><<<blocks, 32 * W, sm, s>>>(jobs, order, njobs, graphs, preps, maxn);
  } else {
    if (sm > 48 * 1024)
      cudaFuncSetAttribute(k_place_list<W, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
    k_place_list<W, false><<<blocks, 32 * W, sm, s>>>(jobs, order, njobs, graphs, preps, maxn);
  }
}

}  // namespace bx

// K2 — the m-ETF / m-SCT list placer for sm_100a.
//
// Restates place_list (proj/src/placers.cpp:115-295) in its exact-argmin
// form (SURVEY.md finding 1): at every step the lexicographic minimum of
// (key(j,p), j, p) over all live (ready, unplaced, not dead, not excluded)
// pairs is either committed or discarded for memory. The reference reaches
// the same sequence through a lazy min-heap with re-pushes (:188-202).
//
// A warp group owns one placement problem for its whole life: a persistent
// scheduling loop, no per-step launches. kW = 1 packs four problems into a
// 128-thread CTA (batched sweeps); kW > 1 gives one large problem a CTA whose
// kW warps split the column rescans (single-graph latency).
//
// Layout:
//   * shared memory (per problem): per-device state — dev_free F, queue
//     tails, reservations, capacities, awake reservations, exclusion flags —
//     and, per device column q, the exact top-KT pairs of that column as a
//     sorted list of (key, node, slot) plus dirty/complete flags;
//   * HBM/L2: ready slots. Kc[q*V + s] holds the key component of the node in
//     slot s on device q (INT64_MAX = discarded pair), column-major so a
//     column rescan is one coalesced 256-byte load per warp instruction.
//     Per in-CSR slot x, pdev[x]/pfin[x] hold the parent's device and finish,
//     written when the parent commits, so keying a node reads its parents in
//     one coalesced level plus the cache probe.
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
// its top list, and new ready rows are merged into the lists.
#include <cstdlib>

#include "sched_common.cuh"

namespace bx {

constexpr int KT = 4;  // exact top-KT pairs kept per device column
#ifndef BX_XR_MODE
// sequential comm, when a rescan keys its column exactly first: 0 never,
// 1 after a re-key dropped an entry, 2 after one emptied the list, 3 always,
// 4 always beyond 4 devices (measured, profiles/r01d_seq_policy.txt)
#define BX_XR_MODE 4
#endif
#ifndef BX_PPC
#define BX_PPC 4  // problems (warps) per warp-kernel CTA
#endif
#ifndef BX_LIST_MINB
#define BX_LIST_MINB 3  // resident 4-problem warp-kernel CTAs per SM (register budget; profiles/r01d_minb.txt)
#endif
#ifndef BX_SCAN_U
#define BX_SCAN_U 4  // column-scan loads in flight per lane, warp kernel
#endif
#ifndef BX_SCAN_U_ROUNDS
#define BX_SCAN_U_ROUNDS 8  // ... round kernel (profiles/r01e_scan_u.txt)
#endif

struct Tops {      // entry k of column q at k * st + q (no bank conflicts for lane-owned columns)
  int64_t *t;    // [KT*st] keys, ascending (key, node)
  int32_t *j;    // [KT*st] nodes
  int32_t *s;    // [KT*st] their ready slots
  int st;
  int32_t *cnt;  // [n]
  int32_t *flg;  // [n] bit0 dirty, bit1 complete (list holds every live pair)
};
constexpr int kDirty = 1, kComplete = 2;

// ---- keys ------------------------------------------------------------------
// schedulable_time_impl (placers.cpp:43-79) for ready node j on device q,
// from the per-slot parent arrays. Parallel mode: data-ready time (t0 = 0).
// Sequential: the full fold through this lane's generation-tagged scratch.
__device__ __forceinline__ int64_t key_of(const Ctx &c, int j, int q, int32_t &gen) {
  const int b = __ldg(c.in_off + (j)), e = __ldg(c.in_off + (j + 1));
  const int n = c.n;
  if (c.mode == 1 && c.nocache) {
    int64_t t = 0;
    for (int x = b; x < e; ++x) {
      const int64_t f = c.pfin[x];
      t = max64(t, c.pdev[x] == q ? f : f + __ldg(c.in_c + (x)));
    }
    return t;
  }
  if (c.mode == 1) {
    int64_t t = 0;
    int x = b;
    for (; x + 1 < e; x += 2) {  // two parents per round: loads issue together
      int d0 = c.pdev[x], d1 = c.pdev[x + 1];
      int64_t f0 = c.pfin[x], f1 = c.pfin[x + 1];
      int i0 = __ldg(c.in_src + (x)), i1 = __ldg(c.in_src + (x + 1));
      int64_t c0 = __ldg(c.in_c + (x)), c1 = __ldg(c.in_c + (x + 1));
      int64_t a0 = d0 == q ? -1 : c.cache[static_cast<int64_t>(i0) * n + q];
      int64_t a1 = d1 == q ? -1 : c.cache[static_cast<int64_t>(i1) * n + q];
      int64_t t0 = d0 == q ? f0 : (a0 >= 0 ? max64(f0, a0) : f0 + c0);
      int64_t t1 = d1 == q ? f1 : (a1 >= 0 ? max64(f1, a1) : f1 + c1);
      t = max64(t, max64(t0, t1));
    }
    if (x < e) {
      int d0 = c.pdev[x];
      int64_t f0 = c.pfin[x];
      int64_t a0 = d0 == q ? -1 : c.cache[static_cast<int64_t>(__ldg(c.in_src + (x))) * n + q];
      t = max64(t, d0 == q ? f0 : (a0 >= 0 ? max64(f0, a0) : f0 + __ldg(c.in_c + (x))));
    }
    return t;
  }
  // sequential comm: the fold on a copy of the tails (placers.cpp:83-91)
  // without the copy — after the first new transfer the copy's tail of q is
  // the running term T and every device it touched holds a value <= T, so a
  // transfer from d starts at max(finish, T, tail[d]) on the LIVE tails
  (void)gen;
  int64_t t = c.F[q];
  int64_t T = c.tail[q];
  for (int x = b; x < e; ++x) {
    const int d = c.pdev[x];
    const int64_t f = c.pfin[x];
    const bool local = d == q;
    const int64_t cached = local ? -1 : c.cache[static_cast<int64_t>(__ldg(c.in_src + (x))) * n + q];
    const bool xfer = !local && cached < 0;
    const int64_t tn = max64(max64(f, T), c.tail[local ? q : d]) + __ldg(c.in_c + (x));
    const int64_t term = local ? f : (xfer ? tn : max64(f, cached));
    T = xfer ? tn : T;
    t = max64(t, term);
  }
  return t;
}

__device__ __forceinline__ int64_t urgency_e(const Ctx &c, int j) {
  int64_t u = 0;
  for (int x = __ldg(c.in_off + (j)); x < __ldg(c.in_off + (j + 1)); ++x) u = max64(u, c.pfin[x] + __ldg(c.in_c + (x)));
  return u;
}

__device__ __forceinline__ int64_t col_key(const Ctx &c, int q, int s, int j) {
  int64_t t = max64(c.Kc[static_cast<int64_t>(q) * c.V + s], c.F[q]);
  if (c.sct) {
    int aw = c.awf[q];
    if (aw >= 0 && aw != j) t = max64(t, min64(c.awu[q], c.urg_s[s]));
  }
  return t;
}

// ---- column scans ------------------------------------------------------------
__device__ __forceinline__ void topk_insert(int64_t (&lt)[KT], int (&lj)[KT], int (&ls)[KT], int64_t t, int j,
                                            int s) {
  if (!lex_less(t, j, lt[KT - 1], lj[KT - 1])) return;
  lt[KT - 1] = t;
  lj[KT - 1] = j;
  ls[KT - 1] = s;
#pragma unroll
  for (int k = KT - 1; k > 0; --k) {
    if (lex_less(lt[k], lj[k], lt[k - 1], lj[k - 1])) {
      int64_t a = lt[k];
      lt[k] = lt[k - 1];
      lt[k - 1] = a;
      int b = lj[k];
      lj[k] = lj[k - 1];
      lj[k - 1] = b;
      b = ls[k];
      ls[k] = ls[k - 1];
      ls[k - 1] = b;
    }
  }
}

// This warp's exact top-KT of column q over slots s0 + lane + k*step < R;
// KT rounds of warp argmin leave the result in lane 0 (dt/dj/ds, cnt) and the
// live-pair count in every lane.
// one device column's scan inputs, by value (the exact fallbacks are not
// inlined, so they must not take the whole context by reference)
struct ColView {
  const int64_t *kcol;
  const int32_t *node_s;
  const int64_t *urg_s;
  int64_t Fq, awu;
  int aw;
};

__device__ __forceinline__ ColView col_view(const Ctx &c, int q) {
  ColView v;
  v.kcol = c.Kc + static_cast<int64_t>(q) * c.V;
  v.node_s = c.node_s;
  v.urg_s = c.urg_s;
  v.Fq = c.F[q];
  v.aw = c.sct ? c.awf[q] : -1;
  v.awu = v.aw >= 0 ? c.awu[q] : 0;
  return v;
}

__device__ __noinline__ void warp_topk_exact(const ColView cv, int s0, int step, int R, int lane, int64_t (&dt)[KT],
                                             int (&dj)[KT], int (&ds)[KT], int &cnt, int &live) {
  int64_t lt[KT];
  int lj[KT], ls[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    lt[k] = kInf;
    lj[k] = INT32_MAX;
    ls[k] = -1;
  }
  live = 0;
  const int64_t *kcol = cv.kcol;
  const int64_t Fq = cv.Fq;
  const int aw = cv.aw;
  const int64_t awu = cv.awu;
  constexpr int U = 4;
  for (int base = s0 + lane; base < R; base += U * step) {
    int64_t kv[U];
    int nd[U];
    int64_t ug[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int s = base + u * step;
      kv[u] = s < R ? kcol[s] : kInf;
      nd[u] = s < R ? cv.node_s[s] : 0;
      ug[u] = (aw >= 0 && s < R) ? cv.urg_s[s] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kv[u] == kInf) continue;
      ++live;
      int64_t t = max64(kv[u], Fq);
      if (aw >= 0 && aw != nd[u]) t = max64(t, min64(awu, ug[u]));
      topk_insert(lt, lj, ls, t, nd[u], base + u * step);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(kFull, live, o);
  cnt = 0;
#pragma unroll
  for (int r = 0; r < KT; ++r) {
    int64_t bt = lt[0];
    unsigned bju = static_cast<unsigned>(lj[0]);
    warp_argmin_u(bt, bju);
    const int64_t bj = static_cast<int>(bju);
    int bs = __shfl_sync(kFull, ls[0], __ffs(__ballot_sync(kFull, lj[0] == bj && lt[0] == bt)) - 1);
    dt[r] = bt;
    dj[r] = static_cast<int>(bj);
    ds[r] = bs;
    if (bt == kInf) break;
    ++cnt;
    if (lj[0] == bj && lt[0] == bt) {  // the owning lane pops its head
#pragma unroll
      for (int k = 0; k < KT - 1; ++k) {
        lt[k] = lt[k + 1];
        lj[k] = lj[k + 1];
        ls[k] = ls[k + 1];
      }
      lt[KT - 1] = kInf;
      lj[KT - 1] = INT32_MAX;
      ls[KT - 1] = -1;
    }
  }
}


// ---- composite-key column scans ----------------------------------------------
// Every key in column q is >= F[q], so (key - F[q]) << 32 | node orders the
// column's pairs (key, node) with ONE 64-bit compare. A key more than 2^32-2
// above F[q] saturates; `clip` reports it and the caller rescans exactly.
constexpr unsigned long long kNoKey = ~0ull;

struct Lane4 {
  unsigned long long k[4];
  int s[4];
  int seen;
  bool clip;
};

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_min_sync(kFull, hi);
  const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
  return (static_cast<unsigned long long>(mhi) << 32) | mlo;
}

// per-lane exact top-4 of this warp's share (slots s0 + lane + k*step < R)
template <int U>
__device__ __forceinline__ void lane_top4(const Ctx &c, int q, int s0, int step, int R, int lane, Lane4 &L) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    L.k[k] = kNoKey;
    L.s[k] = -1;
  }
  L.seen = 0;
  L.clip = false;
  const int64_t *kcol = c.Kc + static_cast<int64_t>(q) * c.V;
  const int64_t Fq = c.F[q];
  const int aw = c.sct ? c.awf[q] : -1;
  const int64_t awu = aw >= 0 ? c.awu[q] : 0;

  for (int base = s0 + lane; base < R; base += U * step) {
    int64_t kv[U];
    int nd[U];
    int64_t ug[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int s = base + u * step;
      kv[u] = s < R ? kcol[s] : kInf;
      nd[u] = s < R ? c.node_s[s] : 0;
      ug[u] = (aw >= 0 && s < R) ? c.urg_s[s] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kv[u] == kInf) continue;
      ++L.seen;
      int64_t t = max64(kv[u], Fq);
      if (aw >= 0 && aw != nd[u]) t = max64(t, min64(awu, ug[u]));
      unsigned long long d = static_cast<unsigned long long>(t - Fq);
      if (d > 0xfffffffeull) {
        L.clip = true;
        d = 0xfffffffeull;
      }
      const unsigned long long ck = (d << 32) | static_cast<unsigned>(nd[u]);
      if (ck < L.k[3]) {
        L.k[3] = ck;
        L.s[3] = base + u * step;
#pragma unroll
        for (int k = 3; k > 0; --k) {
          if (L.k[k] < L.k[k - 1]) {
            const unsigned long long a = L.k[k];
            L.k[k] = L.k[k - 1];
            L.k[k - 1] = a;
            const int b = L.s[k];
            L.s[k] = L.s[k - 1];
            L.s[k - 1] = b;
          }
        }
      }
    }
  }
}

__device__ __forceinline__ void lane4_pop(Lane4 &L) {
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    L.k[k] = L.k[k + 1];
    L.s[k] = L.s[k + 1];
  }
  L.k[3] = kNoKey;
  L.s[3] = -1;
}

// warp_topk_exact's contract through composite keys
__device__ void warp_topk(const Ctx &c, int q, int s0, int step, int R, int lane, int64_t (&dt)[KT],
                          int (&dj)[KT], int (&ds)[KT], int &cnt, int &live) {
  static_assert(KT == 4, "lane lists hold 4");
  Lane4 L;
  lane_top4<BX_SCAN_U>(c, q, s0, step, R, lane, L);
  if (__any_sync(kFull, L.clip)) {
    warp_topk_exact(col_view(c, q), s0, step, R, lane, dt, dj, ds, cnt, live);
    return;
  }
  live = L.seen;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(kFull, live, o);
  const int64_t Fq = c.F[q];
  cnt = 0;
#pragma unroll
  for (int r = 0; r < KT; ++r) {
    const unsigned long long h = warp_min_u64(L.k[0]);
    if (h == kNoKey) {
      dt[r] = kInf;
      dj[r] = INT32_MAX;
      ds[r] = -1;
      break;
    }
    const bool own = L.k[0] == h;
    dt[r] = Fq + static_cast<int64_t>(h >> 32);
    dj[r] = static_cast<int>(h & 0xffffffffull);
    ds[r] = __shfl_sync(kFull, L.s[0], __ffs(__ballot_sync(kFull, own)) - 1);
    ++cnt;
    if (own) lane4_pop(L);
  }
}

// ---- lane-owned list edits (lane q % 32 owns column q) -------------------------
__device__ __forceinline__ void list_remove(const Tops &T, int q, int j) {
  // every entry loaded up front (independent shared-memory loads), then the
  // tail shifted down one place from the removed entry
  const int c = T.cnt[q];
  int64_t lt[KT];
  int lj[KT], ls[KT];
#pragma unroll
  for (int k = 0; k < KT; ++k) {
    lt[k] = T.t[k * T.st + q];
    lj[k] = T.j[k * T.st + q];
    ls[k] = T.s[k * T.st + q];
  }
  int at = -1;
#pragma unroll
  for (int k = 0; k < KT; ++k)
    if (k < c && lj[k] == j) at = k;
  if (at < 0) return;
#pragma unroll
  for (int k = 0; k + 1 < KT; ++k)
    if (k >= at && k + 1 < c) {
      T.t[k * T.st + q] = lt[k + 1];
      T.j[k * T.st + q] = lj[k + 1];
      T.s[k * T.st + q] = ls[k + 1];
    }
  T.cnt[q] = c - 1;
  if (c == 1 && !(T.flg[q] & kComplete)) T.flg[q] |= kDirty;
}

__device__ __forceinline__ void list_insert(const Tops &T, int q, int64_t t, int j, int s) {
  int c = T.cnt[q];
  int f = T.flg[q];
  if (f & kDirty) return;
  if (c == KT) {
    T.flg[q] = f & ~kComplete;  // a live pair now sits outside the list
    if (!lex_less(t, j, T.t[(KT - 1) * T.st + q], T.j[(KT - 1) * T.st + q])) return;
    --c;
  } else if (!(f & kComplete)) {
    // incomplete list: only pairs that beat the last listed one are known
    if (c == 0 || !lex_less(t, j, T.t[(c - 1) * T.st + q], T.j[(c - 1) * T.st + q])) return;
  }
  int k = c;
  while (k > 0 && lex_less(t, j, T.t[(k - 1) * T.st + q], T.j[(k - 1) * T.st + q])) {
    T.t[(k) * T.st + q] = T.t[(k - 1) * T.st + q];
    T.j[(k) * T.st + q] = T.j[(k - 1) * T.st + q];
    T.s[(k) * T.st + q] = T.s[(k - 1) * T.st + q];
    --k;
  }
  T.t[(k) * T.st + q] = t;
  T.j[(k) * T.st + q] = j;
  T.s[(k) * T.st + q] = s;
  T.cnt[q] = c + 1;
}

// bytes of shared memory per device column per problem
constexpr int kSmemPerDevice = 5 * 8 + 2 * KT * 8 + 2 * 4 + 2 * KT * 4 + 4 * 4;
__host__ __device__ constexpr int stage_bytes_per_device(int w) { return w > 1 ? w * (KT * 16 + 4) : 0; }

#define BX_MARK(slot)                 \
  do {                                \
    if (kProf) {                      \
      int64_t now_ = clock64();       \
      prof[slot] += now_ - prof_last; \
      prof_last = now_;               \
    }                                 \
  } while (0)

template <int kW>
__device__ __forceinline__ void group_sync() {
  if (kW > 1) __syncthreads();
  else __syncwarp();
}

// kEtf: compiled for parallel-comm m-ETF only (no sequential queues, no awake
// reservations): a third of the code, which matters when ~28 warps per SM
// run it at unrelated program counters (instruction-fetch stalls).
template <int kW, bool kProf, bool kEtf = false>
__global__ void __launch_bounds__(kW > 1 ? 32 * kW : 32 * BX_PPC, kW > 1 ? 1 : BX_LIST_MINB)
    k_place_list(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                 int maxn, int seq_only) {
  extern __shared__ __align__(16) unsigned char smem[];
  int64_t prof[kProfSlots];
  int64_t prof_last = 0;
  if (kProf) {
#pragma unroll
    for (int k = 0; k < kProfSlots; ++k) prof[k] = 0;
  }
  const int64_t prof_t0 = kProf ? clock64() : 0;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int gw = kW > 1 ? warp : 0;             // warp index inside the problem's group
  const int pslot = kW > 1 ? 0 : warp;          // problem index inside the CTA
  const int slot_id = kW > 1 ? blockIdx.x : blockIdx.x * BX_PPC + warp;
  if (slot_id >= njobs) return;                 // uniform per problem group
  const DJob jb = jobs[order[slot_id]];
  if (jb.skip || jb.algo == 0 || (seq_only && jb.mode == 1)) return;
  if (jb.sdone && *jb.sdone) return;  // placed by the small-frontier kernel (smallsched.cu)
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  // acyclicity then byte-count validation, in the reference's order
  if (g.flags[0] != g.V || g.flags[1]) {
    if (gw == 0 && lane == 0) {
      if (g.flags[0] != g.V) set_err(jb.err, kValidation, E_CYCLE, 0, 0);
      else set_err(jb.err, kValidation, E_NEG_BYTES, 0, 0);
    }
    return;
  }

  Ctx c;
  c.V = g.V;
  c.n = jb.n;
  c.mode = kEtf ? 1 : jb.mode;
  c.sct = kEtf ? false : (jb.algo == 2 && jb.fav != nullptr);
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
  c.nocache = jb.nocache != 0;
  c.finish = jb.finish;
  c.urg_s = jb.urgent;
  c.start = jb.start;
  c.deadc = nullptr;
  c.pending = jb.pending;
  c.alive_s = jb.alive;
  c.node_s = jb.ready;
  c.rpos = jb.rpos;
  c.device_of = jb.device_of;
  c.cseq = jb.cseq;
  c.nc = jb.nc;
  c.scv = jb.sc_val + static_cast<int64_t>(threadIdx.x & (32 * kW - 1)) * jb.n;  // per lane of the group
  c.scg = jb.sc_gen + static_cast<int64_t>(threadIdx.x & (32 * kW - 1)) * jb.n;
  c.pdev = jb.pdev;
  c.pfin = jb.pfin;
  c.inpos = g.inpos;
  Tops T;
  int64_t *stg_t = nullptr;
  int32_t *stg_j = nullptr, *stg_s = nullptr, *stg_live = nullptr;
  // group control words, double-buffered by iteration parity: every warp
  // reads buffer it & 1 after the loop-top barrier, the leader writes the
  // next iteration's values into the other buffer, which nobody can still
  // be reading (they all passed this iteration's barrier)
  int32_t *ctl, *s_R, *s_done, *s_rq;
  int64_t *nk;   // [KT*st] sequential mode: re-keyed list entries
  int32_t *vst;  // [st] sequential mode: commit count + 1 at which the column's list was re-keyed
  int32_t *xr;   // [st] sequential mode: the column's stored keys proved stale -> exact rescan
  {
    const size_t per = static_cast<size_t>(maxn) * (kSmemPerDevice + stage_bytes_per_device(kW)) + 32;  // + control words (2 x 3)
    unsigned char *base = smem + static_cast<size_t>(pslot) * per;
    c.F = reinterpret_cast<int64_t *>(base);
    c.tail = c.F + maxn;
    c.res = c.tail + maxn;
    c.capS = c.res + maxn;
    c.awu = c.capS + maxn;
    T.st = maxn;
    T.t = c.awu + maxn;
    nk = T.t + maxn * KT;
    int64_t *p64 = nk + maxn * KT;
    if (kW > 1) {
      stg_t = p64;
      p64 += static_cast<size_t>(maxn) * kW * KT;
    }
    int32_t *p32 = reinterpret_cast<int32_t *>(p64);
    c.awf = p32;
    c.excl = c.awf + maxn;
    T.j = c.excl + maxn;
    T.s = T.j + maxn * KT;
    T.cnt = T.s + maxn * KT;
    T.flg = T.cnt + maxn;
    vst = T.flg + maxn;
    xr = vst + maxn;
    p32 = xr + maxn;
    if (kW > 1) {
      stg_j = p32;
      stg_s = stg_j + maxn * kW * KT;
      stg_live = stg_s + maxn * kW * KT;
      p32 = stg_live + maxn * kW;
    }
    ctl = p32;  // [2][3]: R, done, the one column the group rescans next (-1: none)
  }
  const int V = c.V, n = c.n;
  const int64_t Vs = V;
  const bool leader = gw == 0;

  if (leader) {
    for (int d = lane; d < n; d += 32) {
      c.F[d] = 0;
      c.tail[d] = 0;
      c.res[d] = 0;
      c.capS[d] = __ldg(c.cap + (d));
      c.awu[d] = 0;
      c.awf[d] = -1;
      c.excl[d] = 0;
      T.cnt[d] = 0;
      T.flg[d] = kDirty;
      vst[d] = 0;
      xr[d] = 0;
    }
    // per-node init + initial ready slots (sources), keys 0 (dev_free = 0)
    int R = 0;
    for (int base = 0; base < V; base += 32) {
      int j = base + lane;
      bool src = false;
      if (j < V) {
        int indeg = __ldg(g.in_off + (j + 1)) - __ldg(g.in_off + (j));
        c.pending[j] = indeg;
        c.device_of[j] = -1;  // (finish times reach the children through pfin: no per-node copy)
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
      for (int s = lane; s < R; s += 32) c.Kc[q * Vs + s] = 0;
    if (lane == 0) {
      ctl[0] = R;
      ctl[1] = V == 0;
      ctl[2] = -1;
    }
  }
  int it = 0;

  int32_t gen = 0;
  int placed = 0, nexcl = 0;
  int64_t discarded = 0, excluded = 0, awake = 0;
  int minptr = 0;  // lane 0 of the leader: first possibly-unplaced slot of need_order
  int err_status = 0, err_code = 0, err_node = 0;
  if (kProf) prof_last = clock64();

  while (true) {
    group_sync<kW>();
    const int32_t *cur = ctl + 3 * (it & 1);
    s_R = ctl + 3 * ((it + 1) & 1);
    s_done = s_R + 1;
    s_rq = s_R + 2;
    ++it;
    if (cur[1]) break;
    int R = cur[0];
    if (leader && lane == 0) {  // carried into the next iteration unless the leader changes them
      s_R[0] = cur[0];
      s_R[1] = cur[1];
      s_R[2] = cur[2];
    }
    if (kProf) ++prof[P_STEPS];
    // ---- rescan the column the leader asked for (every warp of the group) --
    const int rq = cur[2];
    if (rq >= 0) {
      const int qq = rq;
      int64_t dt[KT];
      int dj[KT], ds[KT], cnt, live;
      const bool exact = c.mode == 0 && (BX_XR_MODE == 3 || (BX_XR_MODE == 4 ? n > 4 : xr[qq] != 0));
      if (exact) {
        // sequential comm, a column whose stored keys proved stale: refresh
        // them to exact keys for the current queue tails first (every lane of
        // the group keys its slots with its own scratch), so the rescanned
        // list is exact and its head commits without a re-key
        for (int s2 = gw * 32 + lane; s2 < R; s2 += 32 * kW)
          if (c.Kc[qq * Vs + s2] != kInf) c.Kc[qq * Vs + s2] = key_of(c, c.node_s[s2], qq, gen);
        group_sync<kW>();
      }
      warp_topk(c, qq, gw * 32, 32 * kW, R, lane, dt, dj, ds, cnt, live);
      if (kProf) ++prof[P_RESCANS];
      if (lane == 0) {
        if (kW == 1) {
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            T.t[(k) * T.st + qq] = dt[k];
            T.j[(k) * T.st + qq] = dj[k];
            T.s[(k) * T.st + qq] = ds[k];
          }
          T.cnt[qq] = cnt;
          T.flg[qq] = live <= KT ? kComplete : 0;
          vst[qq] = exact ? placed + 1 : 0;  // exact keys (refreshed above)
          xr[qq] = 0;
        } else {
#pragma unroll
          for (int k = 0; k < KT; ++k) {
            stg_t[gw * KT + k] = k < cnt ? dt[k] : kInf;
            stg_j[gw * KT + k] = k < cnt ? dj[k] : INT32_MAX;
            stg_s[gw * KT + k] = ds[k];
          }
          stg_live[gw] = live;
        }
      }
      if (kW > 1) {
        __syncthreads();
        if (!leader) continue;
        // merge the group's partial lists (kW*KT <= 32 candidates)
        int64_t ct = kInf;
        int cj = INT32_MAX, cs = -1, lv = 0;
        if (lane < kW * KT) {
          ct = stg_t[lane];
          cj = stg_j[lane];
          cs = stg_s[lane];
        }
        if (lane < kW) lv = stg_live[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lv += __shfl_xor_sync(kFull, lv, o);
        int mc = 0;
#pragma unroll
        for (int r = 0; r < KT; ++r) {
          int64_t bt2 = ct;
          unsigned bju2 = static_cast<unsigned>(cj);
          warp_argmin_u(bt2, bju2);
          const int64_t bj2 = static_cast<int>(bju2);
          if (bt2 == kInf) break;
          unsigned own = __ballot_sync(kFull, cj == bj2 && ct == bt2);
          int bs = __shfl_sync(kFull, cs, __ffs(own) - 1);
          if (lane == 0) {
            T.t[(r) * T.st + qq] = bt2;
            T.j[(r) * T.st + qq] = static_cast<int>(bj2);
            T.s[(r) * T.st + qq] = bs;
          }
          ++mc;
          if (cj == bj2 && ct == bt2) {
            ct = kInf;
            cj = INT32_MAX;
          }
        }
        if (lane == 0) {
          T.cnt[qq] = mc;
          T.flg[qq] = lv <= KT ? kComplete : 0;
          vst[qq] = exact ? placed + 1 : 0;  // exact keys (refreshed above)
          xr[qq] = 0;
        }
      }
      if (lane == 0) *s_rq = -1;
    } else if (kW > 1 && !leader) {
      continue;
    }
    __syncwarp();
    BX_MARK(P_RESCAN);

    // ---- leader only from here: argmin over the clean column heads (key,
    // node, device). A dirty column's keys are all >= F[q], so it only has to
    // be rescanned when F[q] does not exceed the best clean head.
    // cell = node * n + device orders (node, device) lexicographically
    int64_t bt = kInf, df = kInf;
    unsigned bi = 0xffffffffu, dq = 0xffffffffu;
    for (int q = lane; q < n; q += 32) {
      if (c.excl[q]) continue;
      if (T.flg[q] & kDirty) {
        if (c.F[q] < df) {  // ascending q per lane: first minimum wins
          df = c.F[q];
          dq = q;
        }
        continue;
      }
      if (T.cnt[q] == 0) continue;
      int64_t t = T.t[q];
      unsigned cell = static_cast<unsigned>(T.j[q]) * static_cast<unsigned>(n) + q;
      if (t < bt || (t == bt && cell < bi)) {
        bt = t;
        bi = cell;
      }
    }
    warp_argmin_u(bt, bi);
    warp_argmin_u(df, dq);
    if (dq != 0xffffffffu && !(bt < df)) {
      if (lane == 0) *s_rq = static_cast<int>(dq);
      __syncwarp();
      BX_MARK(P_ARGMIN);
      continue;
    }
    if (bi == 0xffffffffu) {
      err_status = kInfeasible;
      err_code = E_NO_PAIR;
      if (lane == 0) *s_done = 1;
      continue;
    }
    const int j = static_cast<int>(bi / static_cast<unsigned>(n));
    const int p = static_cast<int>(bi % static_cast<unsigned>(n));
    const int64_t t = bt;
    // the winner's ready slot: parallel m-ETF reads it from rpos, so the
    // lists' slot fields need no relabelling when a slot moves
    const int sj = kEtf ? c.rpos[j] : T.s[p];
    __syncwarp();  // every lane has read the head before any owner edits the lists
    BX_MARK(P_ARGMIN);

    if (c.mode == 0 && vst[p] != placed + 1) {
      // lazy re-key (placers.cpp:198-202). Queue tails only grow, so stored
      // keys are lower bounds and the winner may commit only once its key is
      // exact for the current tails. Batched: the warp re-keys every listed
      // entry of every column not yet re-keyed since the last commit (lanes
      // over (column, entry) items, each with its own scratch tails); then
      // each column's owner keeps the entries that still sort no later than
      // the list's old tail (everything unlisted has a stored key past it,
      // so they stay an exact prefix; the rest drop out with their keys
      // written back, the reference's re-push) and marks the list re-keyed.
      const int items = n * KT;
      for (int it = lane; it < items; it += 32) {
        const int q = it % n, k = it / n;
        if (c.excl[q] || (T.flg[q] & kDirty) || vst[q] == placed + 1 || k >= T.cnt[q]) continue;
        const int x = k * T.st + q;
        const int hj = T.j[x], hs = T.s[x];
        const int64_t fresh = key_of(c, hj, q, gen);
        int64_t key = fresh;
        if (c.sct) {
          const int aw = c.awf[q];
          if (aw >= 0 && aw != hj) key = max64(key, min64(c.awu[q], c.urg_s[hs]));
        }
        nk[x] = key;
        c.Kc[q * Vs + hs] = fresh;
      }
      __syncwarp();
      for (int q = lane; q < n; q += 32) {
        if (c.excl[q] || (T.flg[q] & kDirty) || vst[q] == placed + 1) continue;
        const int cn = T.cnt[q];
        if (cn == 0) continue;
        const bool complete = (T.flg[q] & kComplete) != 0;
        const int64_t ot = T.t[(cn - 1) * T.st + q];
        const int oj = T.j[(cn - 1) * T.st + q];
        int64_t et[KT];
        int ej[KT], es[KT];
        int kept = 0;
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          if (k >= cn) break;
          const int x = k * T.st + q;
          const int64_t t2 = nk[x];
          const int j2 = T.j[x];
          if (complete || !lex_less(ot, oj, t2, j2)) {  // (t2, j2) <= old tail
            int m = kept++;
            while (m > 0 && lex_less(t2, j2, et[m - 1], ej[m - 1])) {
              et[m] = et[m - 1];
              ej[m] = ej[m - 1];
              es[m] = es[m - 1];
              --m;
            }
            et[m] = t2;
            ej[m] = j2;
            es[m] = T.s[x];
          }
        }
#pragma unroll
        for (int k = 0; k < KT; ++k) {
          if (k >= kept) break;
          T.t[k * T.st + q] = et[k];
          T.j[k * T.st + q] = ej[k];
          T.s[k * T.st + q] = es[k];
        }
        T.cnt[q] = kept;
        // stale lower bounds: the column's next rescan keys it exactly
        if (BX_XR_MODE == 1 ? kept < cn : BX_XR_MODE == 2 ? kept == 0 : BX_XR_MODE >= 3) xr[q] = 1;
        if (kept == 0 && !complete) T.flg[q] |= kDirty;
        else vst[q] = placed + 1;
      }
      __syncwarp();
      BX_MARK(P_REKEY);
      continue;
    }
    if (c.mode == 0) BX_MARK(P_REKEY);

    // the winner's metadata and the last ready slot (swap-removed on a
    // commit; nothing before the swap writes it in a commit step), all
    // independent loads issued together
    const int64_t needj = __ldg(c.need + (j)), kj = __ldg(c.k + (j));
    const int ib = __ldg(c.in_off + (j)), ie = __ldg(c.in_off + (j + 1)), ob = __ldg(c.out_off + (j)), oe = __ldg(c.out_off + (j + 1));
    const int last = R - 1;
    int mv = 0;
    int64_t mv_urg = 0, mv_kc = 0;
    int32_t mv_alive = 0;
    if (sj != last) {
      mv = c.node_s[last];
      if (lane == 0) {
        if (!kEtf) mv_urg = c.urg_s[last];
        mv_alive = c.alive_s[last];
      }
      if (lane < n) mv_kc = c.Kc[lane * Vs + last];
    }
    if (c.res[p] + needj > c.capS[p]) {
      // discard (placers.cpp:203-219)
      int left = 0;
      if (lane == 0) {
        c.Kc[p * Vs + sj] = kInf;
        left = --c.alive_s[sj];
      }
      left = __shfl_sync(kFull, left, 0);
      if (left == 0) {
        err_status = kInfeasible;
        err_code = E_FITS_NONE;
        err_node = j;
        if (lane == 0) *s_done = 1;
        continue;
      }
      ++discarded;
      if (lane == (p & 31)) list_remove(T, p, j);
      // smallest need among all unplaced nodes (the `remaining` multiset,
      // placers.cpp:126,208): first unplaced node in ascending-need order
      int64_t minrem = 0;
      if (lane == 0) {
        while (c.device_of[__ldg(g.need_order + (minptr))] >= 0) ++minptr;
        minrem = __ldg(c.need + (__ldg(g.need_order + (minptr))));
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
          if (c.Kc[p * Vs + s] != kInf) {
            c.Kc[p * Vs + s] = kInf;
            if (--c.alive_s[s] == 0) first_dead = min(first_dead, c.node_s[s]);
          }
        }
        if (nexcl == n) {
          for (int x = lane; x < V; x += 32)
            if (c.device_of[x] < 0) first_dead = min(first_dead, x);
        }
        first_dead = warp_min_i32(first_dead);
        if (first_dead != INT32_MAX) {
          err_status = kInfeasible;
          err_code = E_FITS_NONE;
          err_node = first_dead;
          if (lane == 0) *s_done = 1;
          continue;
        }
        if (lane == 0) c.excl[p] = 1;
      }
      __syncwarp();
      BX_MARK(P_DISCARD);
      continue;
    }

    // ---- commit (placers.cpp:221-233) ------------------------------------
    const int64_t fin = t + kj;
    int ncount = 0;
    if (c.mode == 1 && c.nocache) {
      // no cache: nothing to record, no consumer to re-key
    } else if (c.mode == 1) {
      // commit_schedulable_time, parallel mode: every remote uncached parent
      // tensor lands on p at finish + c_e; order-free, so lanes split parents
      for (int x0 = ib; x0 < ie; x0 += 32) {
        int x = x0 + lane;
        bool fresh = false;
        int i = 0;
        if (x < ie) {
          i = __ldg(c.in_src + (x));
          if (c.pdev[x] != p) {
            int64_t *slot = c.cache + static_cast<int64_t>(i) * n + p;
            if (*slot < 0) {
              *slot = c.pfin[x] + __ldg(c.in_c + (x));
              // a producer whose out-edges all carry the same bytes caches
              // finish + the same c its other consumers already use: their
              // keys cannot change, so no re-key (parallel mode only)
              fresh = pr.nu[i] >= 0;
            }
          }
        }
        unsigned m = __ballot_sync(kFull, fresh);
        if (fresh) c.nc[ncount + __popc(m & ((1u << lane) - 1u))] = i;
        ncount += __popc(m);
      }
    } else if (lane == 0) {
      // sequential mode: the fold walks parents in ascending order on the
      // live queue tails (placers.cpp:62-69)
      for (int x = ib; x < ie; ++x) {
        int d = c.pdev[x];
        if (d == p) continue;
        int i = __ldg(c.in_src + (x));
        int64_t *slot = c.cache + static_cast<int64_t>(i) * n + p;
        if (*slot >= 0) continue;
        int64_t term = max64(c.pfin[x], max64(c.tail[d], c.tail[p])) + __ldg(c.in_c + (x));
        c.tail[d] = term;
        c.tail[p] = term;
        *slot = term;
        c.nc[ncount++] = i;
      }
    }
    if (c.mode == 0) ncount = __shfl_sync(kFull, ncount, 0);
    if (lane == 0) {
      c.device_of[j] = p;
      c.start[j] = t;
      c.F[p] = fin;
      c.res[p] += needj;
      c.cseq[placed] = j;
    }
    ++placed;
    if (kProf) ++prof[P_COMMITS];
    BX_MARK(P_COMMIT);
    // swap-remove slot sj: the last slot moves in (lists follow its slot)
    if (sj != last) {
      if (lane < n) c.Kc[lane * Vs + sj] = mv_kc;
      for (int q = lane + 32; q < n; q += 32) c.Kc[q * Vs + sj] = c.Kc[q * Vs + last];
      if (lane == 0) {
        c.node_s[sj] = mv;
        if (!kEtf) c.urg_s[sj] = mv_urg;
        c.alive_s[sj] = mv_alive;
        c.rpos[mv] = sj;
      }
      if (!kEtf) {
#pragma unroll
        for (int k = 0; k < KT; ++k)
          for (int q = lane; q < n; q += 32) {
            const int x = k * T.st + q;
            if (T.j[x] == mv) T.s[x] = sj;
          }
      }
    }
    --R;
    __syncwarp();
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
        int h = __ldg(c.fav + (j));
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

    // ---- readiness (placers.cpp:256-268); publish j to its children's slots
    const int R0 = R;
    for (int base = ob; base < oe; base += 32) {
      int y = base + lane;
      bool fresh = false;
      int child = -1;
      if (y < oe) {
        child = __ldg(c.out_dst + (y));
        int x = __ldg(c.inpos + (y));
        c.pdev[x] = p;
        c.pfin[x] = fin;
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
        if (!kEtf) c.urg_s[s] = c.sct ? urgency_e(c, c.node_s[s]) : 0;  // read only by m-SCT
      }
      for (int r = lane; r < nnew * n; r += 32) {
        int s = R0 + r / n;
        int q = r % n;
        c.Kc[q * Vs + s] = c.excl[q] ? kInf : key_of(c, c.node_s[s], q, gen);
      }
    }
    __syncwarp();
    BX_MARK(P_ROWS);
    // ---- cached parents change their other consumers' keys on p (:271-279)
    for (int a = 0; a < ncount; ++a) {
      int i = c.nc[a];
      for (int y = __ldg(c.out_off + (i)) + lane; y < __ldg(c.out_off + (i + 1)); y += 32) {
        const int cc = __ldg(c.out_dst + (y));
        // the three node loads issue together (no short-circuit chain);
        // rpos is only trusted once the node is known ready and unplaced
        const int pend = c.pending[cc], dv = c.device_of[cc], s = c.rpos[cc];
        if (cc == j || pend != 0 || dv >= 0) continue;
        if (s >= R0) continue;  // new rows were keyed after the cache update
        if (c.Kc[p * Vs + s] == kInf) continue;
        c.Kc[p * Vs + s] = key_of(c, cc, p, gen);
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
          list_insert(T, q, col_key(c, q, s, node), node, s);
        }
      }
    }
    if (lane == 0) {
      *s_R = R;
      if (placed == V) *s_done = 1;
    }
    __syncwarp();
    BX_MARK(P_INSERT);
  }

  if (!leader) return;
  if (err_status) {
    if (lane == 0) set_err(jb.err, err_status, err_code, err_node, 0);
    return;
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

template <int kW, bool kProf, bool kEtf = false>
static void launch_w(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                     int maxn, int seq_only, cudaStream_t s) {
  if (njobs <= 0) return;
  const size_t per = static_cast<size_t>(maxn) * (kSmemPerDevice + stage_bytes_per_device(kW)) + 32;  // + control words (2 x 3)
  const int probs_per_cta = kW > 1 ? 1 : BX_PPC;
  const int threads = kW > 1 ? 32 * kW : 32 * BX_PPC;
  const int blocks = (njobs + probs_per_cta - 1) / probs_per_cta;
  const size_t sm = per * probs_per_cta;
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(k_place_list<kW, kProf, kEtf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sm));
  // the rest of the unified L1/shared array goes to L1: just enough shared
  // memory for the resident CTAs (+3% sweep throughput, profiles/r01d_minb.txt)
  if (kW == 1) {
    int pct = static_cast<int>((100 * size_t(BX_LIST_MINB) * (sm + 1024) + 228 * 1024 - 1) / (228 * 1024)) + 5;
    cudaFuncSetAttribute(k_place_list<kW, kProf, kEtf>, cudaFuncAttributePreferredSharedMemoryCarveout,
                         pct < 100 ? pct : 100);
  }
  k_place_list<kW, kProf, kEtf><<<blocks, threads, sm, s>>>(jobs, order, njobs, graphs, preps, maxn, seq_only);
}

// ============================================================================
// K2r — the round kernel: m-ETF (and m-SCT, one commit per round) in
// parallel comm mode, one problem per 256-thread CTA.
//
// Exactness argument. After committing (j, p) at time t, every key that can
// change or appear is >= t + k_j: column p's keys are >= F[p] = t + k_j, a
// cached parent only touches column p, and a newly ready child has j as a
// parent, so its key is >= finish(j) = t + k_j on every device. Hence, with
// the per-column top lists exact for every column not touched this round,
// the next global argmin is the smallest clean head whose key is strictly
// below min(F[q] over touched ("dirty") columns): it can be committed without
// re-keying anything. A round commits such heads greedily (at most one per
// column), then the whole CTA does the global-memory work of all of them at
// once: cache arrivals, readiness, new key rows, cached-consumer re-keys, and
// the rescans of the touched columns.
// m-SCT: a lifted awake reservation may lower keys in another column, which
// then turns dirty and lowers the round's threshold to its F; discards and
// exclusions are handled inline by the leader.
// ============================================================================
#ifndef BX_RWARPS
#define BX_RWARPS 8
#endif
constexpr int RWARPS = BX_RWARPS;  // warps per round-kernel CTA

struct REnt {
  int64_t t, need, k;
  int32_t j, s, fav, inb, ine, outb, oute, pad;
};

struct RCommit {
  int64_t t, fin;
  int32_t j, q, s, inb, ine, outb, oute, pad;
};

__device__ __forceinline__ void rent_meta(REnt &e, const Ctx &c, const DGraph &g) {
  e.need = __ldg(c.need + (e.j));
  e.k = __ldg(g.k + (e.j));
  e.fav = c.fav ? __ldg(c.fav + (e.j)) : -1;
  e.inb = __ldg(g.in_off + (e.j));
  e.ine = __ldg(g.in_off + (e.j + 1));
  e.outb = __ldg(g.out_off + (e.j));
  e.oute = __ldg(g.out_off + (e.j + 1));
}

// Per-column sorted lists in shared memory, structure of arrays, entry k of
// column q at k * st + q: lanes that own consecutive columns touch consecutive
// words (no bank conflicts for the lane-owned edits and the head scans). The
// sorted order holds (t, j, handle); a node's metadata sits at its handle
// (h * st + q) and never moves, so list edits shift three words, not ten.
struct RList {
  int64_t *t, *need, *k;
  int32_t *j, *h, *s, *fav, *inb, *ine, *outb, *oute;
  int32_t *hmask;  // [st] handles in use per column
  int st;
  __device__ __forceinline__ int at(int q, int kk) const { return kk * st + q; }
  __device__ __forceinline__ REnt get(int q, int kk) const {
    const int i = at(q, kk), m = h[i] * st + q;
    REnt e;
    e.t = t[i];
    e.j = j[i];
    e.need = need[m];
    e.k = k[m];
    e.s = s[m];
    e.fav = fav[m];
    e.inb = inb[m];
    e.ine = ine[m];
    e.outb = outb[m];
    e.oute = oute[m];
    return e;
  }
  __device__ __forceinline__ void put_meta(int q, int hh, const REnt &e) const {
    const int m = hh * st + q;
    need[m] = e.need;
    k[m] = e.k;
    s[m] = e.s;
    fav[m] = e.fav;
    inb[m] = e.inb;
    ine[m] = e.ine;
    outb[m] = e.outb;
    oute[m] = e.oute;
  }
  __device__ __forceinline__ void mv(int d, int x) const {
    t[d] = t[x];
    j[d] = j[x];
    h[d] = h[x];
  }
};

// lane-owned list edits (lane q % 32 owns column q)
template <int KR>
// returns true when the column just turned dirty (emptied, incomplete)
__device__ __forceinline__ bool rlist_remove(const RList &L, int32_t *cnt, int32_t *flg, int q, int j) {
  int c = cnt[q];
  int at = -1;
  for (int k = 0; k < c; ++k)
    if (L.j[L.at(q, k)] == j) at = k;
  if (at < 0) return false;
  L.hmask[q] &= ~(1u << L.h[L.at(q, at)]);
  for (int k = at; k + 1 < c; ++k) L.mv(L.at(q, k), L.at(q, k + 1));
  cnt[q] = --c;
  if (c == 0 && !(flg[q] & kComplete)) {
    flg[q] |= kDirty;
    return true;
  }
  return false;
}

// insert a fully built entry; returns nothing (list stays exact top-cnt)
template <int KR>
__device__ __forceinline__ void rlist_insert(const RList &L, int32_t *cnt, int32_t *flg, int q, const REnt &e) {
  int c = cnt[q];
  int f = flg[q];
  if (f & kDirty) return;
  if (c == KR) {
    flg[q] = f & ~kComplete;
    if (!lex_less(e.t, e.j, L.t[L.at(q, KR - 1)], L.j[L.at(q, KR - 1)])) return;
    --c;
    L.hmask[q] &= ~(1u << L.h[L.at(q, KR - 1)]);  // the dropped tail frees its handle
  } else if (!(f & kComplete)) {
    if (c == 0 || !lex_less(e.t, e.j, L.t[L.at(q, c - 1)], L.j[L.at(q, c - 1)])) return;
  }
  const unsigned used = static_cast<unsigned>(L.hmask[q]);
  const int hh = __ffs(~used) - 1;
  L.hmask[q] = static_cast<int32_t>(used | (1u << hh));
  L.put_meta(q, hh, e);
  int k = c;
  while (k > 0 && lex_less(e.t, e.j, L.t[L.at(q, k - 1)], L.j[L.at(q, k - 1)])) {
    L.mv(L.at(q, k), L.at(q, k - 1));
    --k;
  }
  L.t[L.at(q, k)] = e.t;
  L.j[L.at(q, k)] = e.j;
  L.h[L.at(q, k)] = hh;
  cnt[q] = c + 1;
}

// Exact smallest pairs of column q over this warp's share of the slots
// (s0 + lane + k*step < R). Every lane keeps its own top-LK; a lane that saw
// more than LK live pairs vouches only up to its LK-th pair, so the share's
// sorted order is known exactly up to thr = the least such LK-th pair
// (pairs are unique per column: everything a lane dropped is above it).
// Pops lane heads while <= thr, at most KR, into out_* (lane 0 writes).
template <int KR>
__device__ __noinline__ void warp_prefix_exact(const ColView cv, int s0, int step, int R, int lane, int64_t *out_t,
                                               int32_t *out_j, int32_t *out_s, int &cnt, int64_t &thr_t,
                                               unsigned &thr_j, int &live) {
  constexpr int LK = 4;
  int64_t lt[LK];
  int lj[LK], ls[LK];
#pragma unroll
  for (int k = 0; k < LK; ++k) {
    lt[k] = kInf;
    lj[k] = INT32_MAX;
    ls[k] = -1;
  }
  int seen = 0;
  const int64_t *kcol = cv.kcol;
  const int64_t Fq = cv.Fq;
  const int aw = cv.aw;
  const int64_t awu = cv.awu;
  constexpr int U = 4;
  for (int base = s0 + lane; base < R; base += U * step) {
    int64_t kv[U];
    int nd[U];
    int64_t ug[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      int s = base + u * step;
      kv[u] = s < R ? kcol[s] : kInf;
      nd[u] = s < R ? cv.node_s[s] : 0;
      ug[u] = (aw >= 0 && s < R) ? cv.urg_s[s] : 0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (kv[u] == kInf) continue;
      ++seen;
      int64_t t = max64(kv[u], Fq);
      if (aw >= 0 && aw != nd[u]) t = max64(t, min64(awu, ug[u]));
      topk_insert(lt, lj, ls, t, nd[u], base + u * step);
    }
  }
  int64_t tt = seen > LK ? lt[LK - 1] : kInf;
  unsigned tj = seen > LK ? static_cast<unsigned>(lj[LK - 1]) : 0xffffffffu;
  warp_argmin_u(tt, tj);
  live = seen;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(kFull, live, o);
  cnt = 0;
  int64_t lastt = kInf;
  unsigned lastj = 0xffffffffu;
  for (int r = 0; r < KR; ++r) {
    int64_t bt = lt[0];
    unsigned bju = static_cast<unsigned>(lj[0]);
    warp_argmin_u(bt, bju);
    if (bt == kInf || bt > tt || (bt == tt && bju > tj)) break;
    const bool own = lj[0] == static_cast<int>(bju) && lt[0] == bt;
    if (own) {
      out_t[r] = bt;
      out_j[r] = static_cast<int>(bju);
      out_s[r] = ls[0];
#pragma unroll
      for (int k = 0; k < LK - 1; ++k) {
        lt[k] = lt[k + 1];
        lj[k] = lj[k + 1];
        ls[k] = ls[k + 1];
      }
      lt[LK - 1] = kInf;
      lj[LK - 1] = INT32_MAX;
      ls[LK - 1] = -1;
    }
    lastt = bt;
    lastj = bju;
    ++cnt;
  }
  if (cnt == KR) {  // truncated: the share is exact only up to its last pair
    thr_t = lastt;
    thr_j = lastj;
  } else {
    thr_t = tt;
    thr_j = tj;
  }
}

struct RShared {
  int32_t R, live, placed, done, nnew, nnc, ncommit, ndirty, nexcl, compact;
  int32_t err_status, err_code, err_node, pad;
  int64_t discarded, excluded, awake;
};


// warp_prefix_exact's contract through composite keys
template <int KR>
__device__ void warp_prefix(const Ctx &c, int q, int s0, int step, int R, int lane, int64_t *out_t, int32_t *out_j,
                            int32_t *out_s, int &cnt, int64_t &thr_t, unsigned &thr_j, int &live) {
  Lane4 L;
  lane_top4<BX_SCAN_U_ROUNDS>(c, q, s0, step, R, lane, L);
  if (__any_sync(kFull, L.clip)) {
    warp_prefix_exact<KR>(col_view(c, q), s0, step, R, lane, out_t, out_j, out_s, cnt, thr_t, thr_j, live);
    return;
  }
  unsigned long long thr = warp_min_u64(L.seen > 4 ? L.k[3] : kNoKey);
  live = L.seen;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) live += __shfl_xor_sync(kFull, live, o);
  const int64_t Fq = c.F[q];
  cnt = 0;
  unsigned long long last = kNoKey;
  for (int r = 0; r < KR; ++r) {
    const unsigned long long h = warp_min_u64(L.k[0]);
    if (h == kNoKey || h > thr) break;
    if (L.k[0] == h) {
      out_t[r] = Fq + static_cast<int64_t>(h >> 32);
      out_j[r] = static_cast<int>(h & 0xffffffffull);
      out_s[r] = L.s[0];
      lane4_pop(L);
    }
    last = h;
    ++cnt;
  }
  if (cnt == KR) thr = last;  // truncated: exact only up to its last pair
  if (thr == kNoKey) {
    thr_t = kInf;
    thr_j = 0xffffffffu;
  } else {
    thr_t = Fq + static_cast<int64_t>(thr >> 32);
    thr_j = static_cast<unsigned>(thr & 0xffffffffull);
  }
}

template <int KR>
#ifndef BX_ROUNDS_MINB
#define BX_ROUNDS_MINB 1  // resident round CTAs per SM the register budget allows
#endif
__global__ void __launch_bounds__(RWARPS * 32, BX_ROUNDS_MINB)
    k_place_rounds(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                   int maxn) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tid = threadIdx.x;
  constexpr int NT = RWARPS * 32;
  if (blockIdx.x >= njobs) return;
  const DJob jb = jobs[order[blockIdx.x]];
  if (jb.skip || jb.algo == 0 || jb.mode != 1) return;
  if (jb.sdone && *jb.sdone) return;  // placed by the small-frontier kernel (smallsched.cu)
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  if (g.flags[0] != g.V || g.flags[1]) {
    if (tid == 0) set_err(jb.err, kValidation, g.flags[0] != g.V ? E_CYCLE : E_NEG_BYTES, 0, 0);
    return;
  }
  Ctx c;
  c.V = g.V;
  c.n = jb.n;
  c.mode = 1;
  c.sct = (jb.algo == 2 && jb.fav != nullptr);
  c.k = g.k;
  c.need = g.need;
  c.in_c = pr.in_c;
  c.cap = jb.cap;
  c.in_off = g.in_off;
  c.in_src = g.in_src;
  c.out_off = g.out_off;
  c.out_dst = g.edst;
  c.fav = c.sct ? jb.fav : nullptr;
  c.cmax = *pr.cmax;
  c.Kc = jb.K;
  c.cache = jb.cache;
  c.nocache = jb.nocache != 0;
  c.finish = jb.finish;
  c.urg_s = jb.urgent;
  c.start = jb.start;
  c.deadc = nullptr;
  c.pending = jb.pending;
  c.alive_s = jb.alive;
  c.node_s = jb.ready;
  c.rpos = jb.rpos;
  c.device_of = jb.device_of;
  c.cseq = jb.cseq;
  c.nc = jb.nc;
  c.scv = nullptr;
  c.scg = nullptr;
  c.pdev = jb.pdev;
  c.pfin = jb.pfin;
  c.inpos = g.inpos;
  // double buffers for compaction
  int64_t *Kb = jb.K2, *Ub = jb.urgent2;
  int32_t *Nb = jb.ready2, *Ab = jb.alive2;

  // ---- shared memory --------------------------------------------------------
  const int n = c.n, V = c.V;
  const int64_t Vs = V;
  RShared *S = reinterpret_cast<RShared *>(smem);
  unsigned char *p = smem + ((sizeof(RShared) + 15) & ~size_t(15));
  c.F = reinterpret_cast<int64_t *>(p);
  c.tail = c.F + maxn;  // unused in parallel mode
  c.res = c.tail + maxn;
  c.capS = c.res + maxn;
  c.awu = c.capS + maxn;
  RList L;
  L.st = maxn;
  L.t = c.awu + maxn;
  L.need = L.t + maxn * KR;
  L.k = L.need + maxn * KR;
  RCommit *CM = reinterpret_cast<RCommit *>(L.k + maxn * KR);
  int64_t *stg_t = reinterpret_cast<int64_t *>(CM + maxn);
  const int ntask = maxn > RWARPS ? maxn : RWARPS;
  int64_t *stg_tt = stg_t + ntask * KR;  // per task: threshold of its exact prefix
  int32_t *stg_j = reinterpret_cast<int32_t *>(stg_tt + ntask);
  int32_t *stg_s = stg_j + ntask * KR;
  int32_t *stg_live = stg_s + ntask * KR;
  int32_t *stg_cnt = stg_live + ntask;
  unsigned *stg_tj = reinterpret_cast<unsigned *>(stg_cnt + ntask);
  L.j = reinterpret_cast<int32_t *>(stg_tj + ntask);
  L.h = L.j + maxn * KR;
  L.s = L.h + maxn * KR;
  L.fav = L.s + maxn * KR;
  L.inb = L.fav + maxn * KR;
  L.ine = L.inb + maxn * KR;
  L.outb = L.ine + maxn * KR;
  L.oute = L.outb + maxn * KR;
  L.hmask = L.oute + maxn * KR;
  c.awf = L.hmask + maxn;
  c.excl = c.awf + maxn;
  int32_t *cnt = c.excl + maxn;
  int32_t *flg = cnt + maxn;
  int32_t *dcols = flg + maxn;
  int32_t *inoff = dcols + maxn;    // [maxn+1] prefix of committed in-degrees
  int32_t *outoff = inoff + maxn + 1;  // [maxn+1] prefix of committed out-degrees
  int32_t *wsum = outoff + maxn + 1;  // [RWARPS+1] compaction prefix

  // ---- init -------------------------------------------------------------------
  if (tid == 0) {
    S->R = 0;
    S->live = 0;
    S->placed = 0;
    S->done = V == 0;
    S->nnew = 0;
    S->nnc = 0;
    S->ncommit = 0;
    S->nexcl = 0;
    S->compact = 0;
    S->err_status = 0;
    S->discarded = S->excluded = S->awake = 0;
  }
  for (int d = tid; d < n; d += NT) {
    c.F[d] = 0;
    c.res[d] = 0;
    c.capS[d] = __ldg(c.cap + (d));
    c.awu[d] = 0;
    c.awf[d] = -1;
    c.excl[d] = 0;
    cnt[d] = 0;
    flg[d] = kDirty;
  }
  __syncthreads();
  for (int j = tid; j < V; j += NT) {
    int indeg = __ldg(g.in_off + (j + 1)) - __ldg(g.in_off + (j));
    c.pending[j] = indeg;
    c.device_of[j] = -1;
    c.rpos[j] = -1;  // read speculatively beside pending / device_of (the cached-consumer re-keys)
    if (indeg == 0) {
      int s = atomicAdd(&S->R, 1);
      c.node_s[s] = j;
      c.rpos[j] = s;
      c.urg_s[s] = 0;
      c.alive_s[s] = n;
    }
  }
  __syncthreads();
  {
    const int R = S->R;
    for (int64_t x = tid; x < static_cast<int64_t>(R) * n; x += NT) c.Kc[(x / R) * Vs + (x % R)] = 0;
    if (tid == 0) {
      S->live = R;
      S->ndirty = 0;
      for (int q = 0; q < n; ++q) dcols[S->ndirty++] = q;
    }
  }
  int minptr = 0;  // tid 0 only
  // latency breakdown (BX_PROFILE builds): thread 0 charges phase cycles
  const bool prof = jb.prof != nullptr;
  int64_t pc[kProfSlots];
  for (int i = 0; i < kProfSlots; ++i) pc[i] = 0;
  int64_t plast = clock64();
  const int64_t pt0 = plast;
#define RMARK(slot)                    \
  do {                                 \
    if (prof && tid == 0) {            \
      int64_t now_ = clock64();        \
      pc[slot] += now_ - plast;        \
      plast = now_;                    \
    }                                  \
  } while (0)

  while (true) {
    __syncthreads();
    if (S->done) break;
    if (prof && tid == 0) ++pc[P_STEPS];
    // ---- compaction of committed (hole) slots, rarely --------------------------
    if (S->compact) {
      const int R = S->R;
      const int chunk = (R + RWARPS - 1) / RWARPS;
      const int lo = warp * chunk, hi = min(R, lo + chunk);
      int mine = 0;
      for (int b = lo; b < hi; b += 32) {
        int s = b + lane;
        bool keep = s < hi && c.device_of[c.node_s[s]] < 0;
        mine += __popc(__ballot_sync(kFull, keep));
      }
      if (lane == 0) wsum[warp + 1] = mine;
      __syncthreads();
      if (tid == 0) {
        wsum[0] = 0;
        for (int w = 0; w < RWARPS; ++w) wsum[w + 1] += wsum[w];
      }
      __syncthreads();
      int base = wsum[warp];
      for (int b = lo; b < hi; b += 32) {
        int s = b + lane;
        bool keep = s < hi && c.device_of[c.node_s[s]] < 0;
        unsigned m = __ballot_sync(kFull, keep);
        if (keep) {
          int to = base + __popc(m & ((1u << lane) - 1u));
          int node = c.node_s[s];
          Nb[to] = node;
          Ub[to] = c.urg_s[s];
          Ab[to] = c.alive_s[s];
          c.rpos[node] = to;
          for (int q = 0; q < n; ++q) Kb[q * Vs + to] = c.Kc[q * Vs + s];
        }
        base += __popc(m);
      }
      __syncthreads();
      // last round's new rows follow their nodes (inserted after the rescans)
      for (int r = tid; r < S->nnew; r += NT) jb.newl[r] = c.rpos[c.node_s[jb.newl[r]]];
      __syncthreads();
      // swap buffers (every thread keeps its own copy of the pointers)
      int64_t *tK = c.Kc;
      c.Kc = Kb;
      Kb = tK;
      int64_t *tU = c.urg_s;
      c.urg_s = Ub;
      Ub = tU;
      int32_t *tN = c.node_s;
      c.node_s = Nb;
      Nb = tN;
      int32_t *tA = c.alive_s;
      c.alive_s = Ab;
      Ab = tA;
      if (tid == 0) {
        S->R = wsum[RWARPS];
        S->compact = 0;
      }
      // list entries follow their nodes
      for (int e = tid; e < maxn * KR; e += NT)
        if (e % maxn < n && e / maxn < cnt[e % maxn]) L.s[L.h[e] * maxn + e % maxn] = c.rpos[L.j[e]];
      __syncthreads();
      RMARK(P_REMOVE);
    }
    const int R = S->R;
    // ---- phase D: rescans of dirty columns, split over the 8 warps ------------
    const int nd = S->ndirty;
    if (nd > 0) {
      const int parts = nd >= RWARPS ? 1 : RWARPS / nd;
      for (int task = warp; task < nd * parts; task += RWARPS) {
        const int q = dcols[task / parts], part = task % parts;
        int kc, live;
        int64_t tt;
        unsigned tj;
        warp_prefix<KR>(c, q, part * 32, 32 * parts, R, lane, stg_t + task * KR, stg_j + task * KR,
                        stg_s + task * KR, kc, tt, tj, live);
        if (lane == 0) {
          stg_cnt[task] = kc;
          stg_live[task] = live;
          stg_tt[task] = tt;
          stg_tj[task] = tj;
        }
      }
      __syncthreads();
      for (int ci = warp; ci < nd; ci += RWARPS) {
        const int q = dcols[ci];
        // merge the parts' exact prefixes up to the least threshold
        const int tb = ci * parts;
        int ptr = 0, cl = 0, lv = 0;
        int64_t thr_t = kInf;
        unsigned thr_j = 0xffffffffu;
        if (lane < parts) {
          cl = stg_cnt[tb + lane];
          lv = stg_live[tb + lane];
          thr_t = stg_tt[tb + lane];
          thr_j = stg_tj[tb + lane];
        }
        warp_argmin_u(thr_t, thr_j);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) lv += __shfl_xor_sync(kFull, lv, o);
        int kc = 0;
        for (int r = 0; r < KR; ++r) {
          const bool has = lane < parts && ptr < cl;
          const int64_t ht = has ? stg_t[(tb + lane) * KR + ptr] : kInf;
          const unsigned hj = has ? static_cast<unsigned>(stg_j[(tb + lane) * KR + ptr]) : 0xffffffffu;
          int64_t bt = ht;
          unsigned bj = hj;
          warp_argmin_u(bt, bj);
          if (bt == kInf || bt > thr_t || (bt == thr_t && bj > thr_j)) break;
          if (has && ht == bt && hj == bj) {
            L.t[L.at(q, r)] = bt;
            L.j[L.at(q, r)] = static_cast<int>(bj);
            L.h[L.at(q, r)] = r;
            L.s[L.at(q, r)] = stg_s[(tb + lane) * KR + ptr];  // handle r: meta row r
            ++ptr;
          }
          ++kc;
        }
        __syncwarp();
        for (int r = lane; r < kc; r += 32) {  // listed nodes' metadata, in parallel
          REnt e;
          e.j = L.j[L.at(q, r)];
          e.s = L.s[L.at(q, r)];
          rent_meta(e, c, g);
          L.put_meta(q, r, e);
        }
        if (lane == 0) {
          cnt[q] = kc;
          flg[q] = lv == kc ? kComplete : 0;
          L.hmask[q] = static_cast<int32_t>(kc >= 32 ? 0xffffffffu : (1u << kc) - 1u);
        }
      }
    }
    if (prof && tid == 0) pc[P_RESCANS] += nd;
    RMARK(P_RESCAN);
    // new rows of the last round join the clean lists (dirty ones were rescanned)
    const int nnew = S->nnew;
    if (nnew > 0) {
      for (int q = warp; q < n; q += RWARPS) {
        bool wasdirty = false;  // rescanned this phase: already includes the new rows
        for (int ci = 0; ci < nd; ++ci) wasdirty |= dcols[ci] == q;
        if (wasdirty || c.excl[q] || (flg[q] & kDirty)) continue;
        for (int r0 = 0; r0 < nnew; r0 += 32) {
          REnt e;
          bool have = r0 + lane < nnew;
          if (have) {
            e.s = jb.newl[r0 + lane];
            e.j = c.node_s[e.s];
            e.t = col_key(c, q, e.s, e.j);
            rent_meta(e, c, g);
          }
          for (int l = 0; l < 32 && r0 + l < nnew; ++l) {
            REnt x;
            x.t = __shfl_sync(kFull, e.t, l);
            x.need = __shfl_sync(kFull, e.need, l);
            x.k = __shfl_sync(kFull, e.k, l);
            x.j = __shfl_sync(kFull, e.j, l);
            x.s = __shfl_sync(kFull, e.s, l);
            x.fav = __shfl_sync(kFull, e.fav, l);
            x.inb = __shfl_sync(kFull, e.inb, l);
            x.ine = __shfl_sync(kFull, e.ine, l);
            x.outb = __shfl_sync(kFull, e.outb, l);
            x.oute = __shfl_sync(kFull, e.oute, l);
            if (lane == 0 && x.t != kInf) rlist_insert<KR>(L, cnt, flg, q, x);
          }
        }
      }
    }
    __syncthreads();
    RMARK(P_INSERT);

    // ---- phase S: the leader selects this round's commits (shared memory) -------
    if (warp == 0) {
      int k = 0;
      // threshold: keys in dirty columns are >= F[q]; a commit lowers it to
      // its finish (its column turns dirty), nothing in the round raises it
      // except an exclusion, where the stale lower value is only conservative
      int64_t thr = kInf;
      {
        unsigned dummy = 0;
        for (int q = lane; q < n; q += 32)
          if (!c.excl[q] && (flg[q] & kDirty)) thr = min64(thr, c.F[q]);
        warp_argmin_u(thr, dummy);
      }
      while (true) {
        if (S->placed + k == V) break;
        int64_t bt = kInf;
        unsigned bi = 0xffffffffu;
        for (int q = lane; q < n; q += 32) {
          if (c.excl[q] || (flg[q] & kDirty)) continue;
          if (cnt[q] == 0) continue;
          unsigned cell = static_cast<unsigned>(L.j[q]) * static_cast<unsigned>(n) + q;
          if (L.t[q] < bt || (L.t[q] == bt && cell < bi)) {
            bt = L.t[q];
            bi = cell;
          }
        }
        warp_argmin_u(bt, bi);
        RMARK(P_REKEY);  // (profile builds) phase S: head argmin
        if (bi == 0xffffffffu) {
          if (k == 0 && thr == kInf) {  // no live pair anywhere
            if (lane == 0) {
              S->err_status = kInfeasible;
              S->err_code = E_NO_PAIR;
              S->done = 1;
            }
          }
          break;
        }
        if (bt >= thr) break;
        const int q = static_cast<int>(bi % static_cast<unsigned>(n));
        const REnt e = L.get(q, 0);
        if (c.res[q] + e.need > c.capS[q]) {
          // discard (placers.cpp:203-219), inline: rare. With commits pending
          // in this round, end the round first: the pair stays the minimum
          // (every key the round adds is above it), and the exclusion scan
          // must not see half-committed nodes.
          if (k > 0) break;
          int left = 0;
          if (lane == 0) {
            c.Kc[q * Vs + e.s] = kInf;
            left = --c.alive_s[e.s];
          }
          left = __shfl_sync(kFull, left, 0);
          if (left == 0) {
            if (lane == 0) {
              S->err_status = kInfeasible;
              S->err_code = E_FITS_NONE;
              S->err_node = e.j;
              S->done = 1;
            }
            break;
          }
          if (lane == 0) S->discarded++;
          const bool emptied = lane == (q & 31) && rlist_remove<KR>(L, cnt, flg, q, e.j);
          if (__any_sync(kFull, emptied)) thr = min64(thr, c.F[q]);  // its keys are >= F[q]
          int64_t minrem = 0;
          if (lane == 0) {
            while (c.device_of[__ldg(g.need_order + (minptr))] >= 0) ++minptr;
            minrem = __ldg(c.need + (__ldg(g.need_order + (minptr))));
          }
          minrem = __shfl_sync(kFull, minrem, 0);
          if (c.res[q] + minrem > c.capS[q]) {
            int ne = 0;
            if (lane == 0) {
              S->excluded++;
              ne = ++S->nexcl;
            }
            ne = __shfl_sync(kFull, ne, 0);
            int first_dead = INT32_MAX;
            for (int s = lane; s < R; s += 32) {
              int nd2 = c.node_s[s];
              if (c.device_of[nd2] >= 0) continue;  // committed (hole) slot
              if (c.Kc[q * Vs + s] != kInf) {
                c.Kc[q * Vs + s] = kInf;
                if (--c.alive_s[s] == 0) first_dead = min(first_dead, nd2);
              }
            }
            if (ne == n) {
              for (int x = lane; x < V; x += 32)
                if (c.device_of[x] < 0) first_dead = min(first_dead, x);
            }
            first_dead = warp_min_i32(first_dead);
            if (first_dead != INT32_MAX) {
              if (lane == 0) {
                S->err_status = kInfeasible;
                S->err_code = E_FITS_NONE;
                S->err_node = first_dead;
                S->done = 1;
              }
              break;
            }
            if (lane == 0) c.excl[q] = 1;
          }
          __syncwarp();
          continue;
        }
        RMARK(P_READY);  // (profile builds) phase S: candidate fetch + memory test
        // commit (placers.cpp:221-233): bookkeeping here, global work below
        const int64_t fin = e.t + e.k;
        if (lane == 0) {
          RCommit &cm = CM[k];
          cm.t = e.t;
          cm.fin = fin;
          cm.j = e.j;
          cm.q = q;
          cm.s = e.s;
          cm.inb = e.inb;
          cm.ine = e.ine;
          cm.outb = e.outb;
          cm.oute = e.oute;
          c.F[q] = fin;
          c.res[q] += e.need;
        }
        thr = min64(thr, fin);
        ++k;
        __syncwarp();
        {
          int64_t te = kInf;  // columns emptied by the removal turn dirty too
          for (int qq = lane; qq < n; qq += 32) {
            if (qq == q) flg[qq] |= kDirty;
            else if (rlist_remove<KR>(L, cnt, flg, qq, e.j) && !c.excl[qq]) te = min64(te, c.F[qq]);
          }
          if (__any_sync(kFull, te != kInf)) {
            unsigned dummy = 0;
            warp_argmin_u(te, dummy);
            thr = min64(thr, te);
          }
        }
        __syncwarp();
        RMARK(P_CACHE);  // (profile builds) phase S: bookkeeping + list removals
        if (c.sct) {
          // awake reservations (placers.cpp:235-254). A lifted reservation
          // can lower keys in its column: that column turns dirty and lowers
          // the threshold to its F (its keys stay >= F), so the round goes
          // on exactly; a new reservation only touches column q (dirty).
          // h is j's child, so it cannot have committed earlier this round.
          int64_t tl = kInf;
          if (lane == 0) {
            c.awf[q] = -1;
            for (int qq = 0; qq < n; ++qq)
              if (c.awf[qq] == e.j) {
                c.awf[qq] = -1;
                flg[qq] |= kDirty;
                if (!c.excl[qq]) tl = min64(tl, c.F[qq]);
              }
            int h = e.fav;
            if (h >= 0 && c.device_of[h] < 0) {
              c.awf[q] = h;
              c.awu[q] = fin + c.cmax;
              S->awake++;
            }
          }
          thr = min64(thr, __shfl_sync(kFull, tl, 0));
          __syncwarp();
        }
      }
      // only dirty columns that could beat the best clean head get rescanned
      // (their keys are all >= F[q]); the others stay dirty, lists stale
      int64_t tb = kInf;
      for (int q = lane; q < n; q += 32)
        if (!c.excl[q] && !(flg[q] & kDirty) && cnt[q] > 0) tb = min64(tb, L.t[q]);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) tb = min64(tb, __shfl_xor_sync(kFull, tb, o));
      // prefix sums of the committed nodes' degrees; dirty column list
      {
        int ci = 0, co = 0;
        for (int b = 0; b < k; b += 32) {
          const int i = b + lane;
          int vi = i < k ? CM[i].ine - CM[i].inb : 0, vo = i < k ? CM[i].oute - CM[i].outb : 0;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int ui = __shfl_up_sync(kFull, vi, o), uo = __shfl_up_sync(kFull, vo, o);
            if (lane >= o) {
              vi += ui;
              vo += uo;
            }
          }
          if (i < k) {
            inoff[i + 1] = ci + vi;
            outoff[i + 1] = co + vo;
          }
          ci += __shfl_sync(kFull, vi, 31);
          co += __shfl_sync(kFull, vo, 31);
        }
        if (lane == 0) {
          S->ncommit = k;
          inoff[0] = outoff[0] = 0;
          S->nnew = 0;
          S->nnc = 0;
        }
      }
      {
        int ndc = 0;
        for (int q0 = 0; q0 < n; q0 += 32) {
          const int q = q0 + lane;
          const bool want = q < n && (flg[q] & kDirty) && !c.excl[q] && !(tb < c.F[q]);
          const unsigned m = __ballot_sync(kFull, want);
          if (want) dcols[ndc + __popc(m & ((1u << lane) - 1u))] = q;
          ndc += __popc(m);
        }
        if (lane == 0) S->ndirty = ndc;
      }
      RMARK(P_DISCARD);  // (profile builds) phase S: round tail
    }
    __syncthreads();
    RMARK(P_ARGMIN);
    if (S->done && S->err_status) break;
    const int kc = S->ncommit;
    if (prof && tid == 0) pc[P_COMMITS] += kc;
    const int placed0 = S->placed;
    // ---- phase B: commit bookkeeping, cache arrivals, readiness (all warps) -----
    for (int i = warp; i < kc; i += RWARPS) {
      const RCommit cm = CM[i];
      if (lane == 0) {
        c.device_of[cm.j] = cm.q;
        c.start[cm.j] = cm.t;
        c.finish[cm.j] = cm.fin;
        c.cseq[placed0 + i] = cm.j;
      }
      for (int q = lane; q < n; q += 32) c.Kc[q * Vs + cm.s] = kInf;  // slot becomes a hole
    }
    {
      const int nin = inoff[kc];
      for (int w = tid; w < nin; w += NT) {
        int i = 0;
        while (inoff[i + 1] <= w) ++i;
        const RCommit &cm = CM[i];
        const int x = cm.inb + (w - inoff[i]);
        if (!c.nocache && c.pdev[x] != cm.q) {
          const int par = __ldg(c.in_src + (x));
          int64_t *slot = c.cache + static_cast<int64_t>(par) * n + cm.q;
          if (*slot < 0) {  // commit_schedulable_time, parallel mode
            *slot = c.pfin[x] + __ldg(c.in_c + (x));
            if (pr.nu[par] >= 0) {  // uniform producers change no consumer key (see the warp kernel)
              int a = atomicAdd(&S->nnc, 1);
              c.nc[a] = par;
              jb.ncw[a] = i;
            }
          }
        }
      }
      const int nout = outoff[kc];
      for (int w = tid; w < nout; w += NT) {
        int i = 0;
        while (outoff[i + 1] <= w) ++i;
        const RCommit &cm = CM[i];
        const int y = cm.outb + (w - outoff[i]);
        const int child = __ldg(c.out_dst + (y));
        const int x = __ldg(c.inpos + (y));
        c.pdev[x] = cm.q;
        c.pfin[x] = cm.fin;
        __threadfence_block();
        if (atomicSub(&c.pending[child], 1) == 1) {
          int s = atomicAdd(&S->R, 1);
          c.node_s[s] = child;
          c.rpos[child] = s;
          jb.newl[atomicAdd(&S->nnew, 1)] = s;
        }
      }
    }
    __syncthreads();
    RMARK(P_COMMIT);
    // ---- phase C: new key rows + cached-consumer re-keys (all warps) ------------
    {
      const int nn = S->nnew;
      const int nexcl = S->nexcl;
      const int Rnow = S->R;
      const int R0 = Rnow - nn;
      int32_t gen = 0;
      for (int64_t w = tid; w < static_cast<int64_t>(nn) * n; w += NT) {
        const int r = static_cast<int>(w / n), q = static_cast<int>(w % n);
        const int s = jb.newl[r];
        const int ch = c.node_s[s];
        c.Kc[q * Vs + s] = c.excl[q] ? kInf : key_of(c, ch, q, gen);
        if (q == 0) {
          c.alive_s[s] = n - nexcl;
          c.urg_s[s] = c.sct ? urgency_e(c, ch) : 0;
        }
      }
      const int nnc = S->nnc;
      for (int a = warp; a < nnc; a += RWARPS) {
        const int par = c.nc[a];
        const int q = CM[jb.ncw[a]].q;
        for (int y = __ldg(g.out_off + (par)) + lane; y < __ldg(g.out_off + (par + 1)); y += 32) {
          const int cc = __ldg(c.out_dst + (y));
          const int pend = c.pending[cc], dv = c.device_of[cc], s = c.rpos[cc];  // issued together
          if (pend != 0 || dv >= 0) continue;
          if (s >= R0) continue;  // new rows were keyed after the cache update
          if (c.Kc[q * Vs + s] == kInf) continue;
          c.Kc[q * Vs + s] = key_of(c, cc, q, gen);
        }
      }
      if (tid == 0) {
        S->placed += kc;
        S->live += nn - kc;
        if (S->placed == V) S->done = 1;
        // holes dominate the slot range: compact next round
        if (S->R - S->live > 1024 && S->R - S->live > S->live) S->compact = 1;
      }
    }
    RMARK(P_ROWS);
  }
  __syncthreads();
  if (warp != 0) return;
  if (S->err_status) {
    if (lane == 0) set_err(jb.err, S->err_status, S->err_code, S->err_node, 0);
    return;
  }
  emit_exec_order(c, jb, c.excl, lane);
  if (lane == 0) {
    jb.stats[0] = S->discarded;
    jb.stats[1] = S->excluded;
    jb.stats[2] = S->awake;
    set_err(jb.err, kOk, E_NONE, 0, 0);
    if (prof) {
      pc[P_TOTAL] = clock64() - pt0;
      for (int i = 0; i < kProfSlots; ++i) jb.prof[i] = pc[i];
    }
  }
#undef RMARK
}

static size_t rounds_smem(int maxn, int KR) {
  const int ntask = maxn > RWARPS ? maxn : RWARPS;
  return ((sizeof(RShared) + 15) & ~size_t(15)) + 5 * 8 * size_t(maxn) + 56 * size_t(KR) * maxn + 4 * size_t(maxn) +
         sizeof(RCommit) * maxn + size_t(ntask) * (KR * 16 + 8 + 12) +
         4 * (7 * size_t(maxn) + 2) + 4 * (RWARPS + 1) + 64;  // awf excl cnt flg dcols inoff outoff wsum
}

template <int KR>
static void launch_rounds_kr(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs,
                             const DPrep *preps, int maxn, cudaStream_t s) {
  const size_t sm = rounds_smem(maxn, KR);
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(k_place_rounds<KR>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(sm));
  k_place_rounds<KR><<<njobs, RWARPS * 32, sm, s>>>(jobs, order, njobs, graphs, preps, maxn);
}

// List length per device column. The columns' heads are largely the same
// nodes, so with many devices short lists drain together and every column
// needs a rescan every few commits; with few devices each commit rescans just
// its own column and longer lists only cost more per rescan and per edit
// (measured, profiles/r01c_kr_sweep.txt, r01e_scan_u.txt): 4 up to 8
// devices, 8 up to 31, 16 up to 47, 32 (100k x 64: 1.27 -> 1.07 s vs 16).
void launch_rounds(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                   int maxn, int list_len, cudaStream_t s) {
  int kr = maxn <= 8 ? 4 : maxn < 32 ? 8 : maxn < 48 ? 16 : 32;
  if (list_len > 0) kr = list_len;  // bx_plan_options.list_len (tests drive every length)
  while (kr > 4 && rounds_smem(maxn, kr) > 200 * 1024) kr /= 2;
  if (kr >= 32) launch_rounds_kr<32>(jobs, order, njobs, graphs, preps, maxn, s);
  else if (kr >= 16) launch_rounds_kr<16>(jobs, order, njobs, graphs, preps, maxn, s);
  else if (kr >= 8) launch_rounds_kr<8>(jobs, order, njobs, graphs, preps, maxn, s);
  else launch_rounds_kr<4>(jobs, order, njobs, graphs, preps, maxn, s);
}


// Launch lists come from bx_plan_create: small problems one warp each (the
// first n_etf of them parallel-comm m-ETF, on the specialised kernel),
// big sequential-mode problems an 8-warp CTA each.
void launch_small(const DJob *jobs, const int32_t *order, int n_etf, int n_gen, const DGraph *graphs,
                  const DPrep *preps, int maxn, bool prof, cudaStream_t s, cudaStream_t s_gen) {
  if (prof) {
    launch_w<1, true, true>(jobs, order, n_etf, graphs, preps, maxn, 0, s);
    launch_w<1, true>(jobs, order + n_etf, n_gen, graphs, preps, maxn, 0, s_gen);
  } else {
    launch_w<1, false, true>(jobs, order, n_etf, graphs, preps, maxn, 0, s);
    launch_w<1, false>(jobs, order + n_etf, n_gen, graphs, preps, maxn, 0, s_gen);
  }
}

void launch_big_seq(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                    int maxn, bool prof, cudaStream_t s) {
  if (prof) launch_w<8, true>(jobs, order, njobs, graphs, preps, maxn, 0, s);
  else launch_w<8, false>(jobs, order, njobs, graphs, preps, maxn, 0, s);
}

}  // namespace bx

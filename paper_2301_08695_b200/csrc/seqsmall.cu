// K2q — the small-frontier list placer for SEQUENTIAL comm mode (m-ETF).
//
// Same contract as K2 / K2s (place_list, proj/src/placers.cpp:115-295, in its
// exact-argmin form): every step takes the lexicographic minimum of
// (schedulable_time(j, p), j, p) over the live pairs and commits or discards
// it. Sequential comm serialises every transfer through per-device queue
// tails (placers.cpp:62-68), and a commit that moves a tensor moves two tails,
// so one commit can change the key of every live pair. The general kernels
// keep stored lower bounds and re-key lazily (the reference's heap does the
// same); on graphs whose ready frontier is a handful of nodes (the
// reference's own layered-chain family) that bookkeeping costs more than
// recomputing every live key. This kernel does exactly that, one warp per
// problem, no CTA barriers:
//
//   1. keys + selection in one pass: every live (slot, device) pair (<= 512,
//      lanes stride the pair index) folds its parents in ascending in-edge
//      order (placers.cpp:43-79) — the first 8 parents' (index, device,
//      finish, comm time) recorded in shared memory when the slot became
//      ready (fixed from then on; only the cache and the tails move), the
//      cache arrival read from the job's K array (L1/L2-resident). The fold
//      needs no scratch copy of the tails: after the first uncached remote
//      parent the scratch tail of p is the running term T, and every device
//      touched since holds a value <= T, so the queue start of the next
//      transfer from q is max(finish_i, T, tail[q]) with the LIVE tail[q].
//      Then two REDUX for the 64-bit key, one for (node << 5 | device); the
//      owner lane names the winner's slot;
//   2. discard (placers.cpp:203-219) or commit: the winner's key fold ran on
//      exactly the state the commit sees, so it doubles as the commit recipe
//      (its new transfers: parent, device, arrival) and the winner's lane
//      stores the tails and cache arrivals (commit_schedulable_time,
//      :95-101; a cache row is initialised when its producer commits; more
//      than two transfers: lane 0 replays the fold), dev_free / reserved /
//      outputs;
//   3. readiness of the children (:256-268): the slot's first 8 children
//      were cached when it became ready; pending counts are bytes in shared
//      memory when they fit (one warp owns them; meta edges are unique), else
//      the job's HBM array with atomics issued before the commit; the new
//      slots' records load in one level of independent reads past the node's
//      offsets.
// The per-parent step is branch-free: lanes hold pairs whose parents take
// different cases, and a branchy fold made the warp issue every case's path.
// Measured and rejected (the reference's layered-chain 100k x 4, sequential
// comm): several commits per round while a commit moves no queue tail (1.33
// commits per round there), cache arrivals mirrored into the slot records, a
// shared-memory table of recent producers' cache rows, the children's node
// fields recorded with their parent's slot, L1 prefetches of them each step
// (K2q).
//
// Times stay int64 (no range checks). Eligibility (checked on the device):
// acyclic, non-negative byte counts and compute times, comm times in
// [0, 2^16) (the prep's check), at most 32 devices, fewer than 2^26 nodes,
// and a frontier of at most 512 pairs at every step; anything else leaves
// sdone = 0 and the general kernels, launched behind this one, place the job
// from scratch (they re-initialise every per-node array this kernel touched;
// the cache they read is not written here).
#include "sched_common.cuh"

namespace bx {

constexpr int kQPairs = 512;  // live pairs per problem
constexpr int kQKI = 8;       // parents recorded per ready slot (the rest read from the graph)
constexpr int kQKO = 8;       // children recorded per ready slot
constexpr int kQWarps = 8;    // CTA size for the init; warp 0 alone schedules
constexpr int kQPendV = 160 * 1024;  // largest graph whose pending counts live in shared memory
constexpr size_t kQSmemMax = 220 * 1024;  // dynamic shared memory per CTA

__host__ __device__ inline int seq_small_slots(int n) { return kQPairs / (n > 0 ? n : 1); }

__host__ __device__ inline size_t seq_small_smem_bytes(int n) {
  const size_t ns = static_cast<size_t>(seq_small_slots(n));
  return 4 * 32 * 8 + 32 * 4 + 16                    // F, tail, res, cap; exec counters; control
         + ns * (8 + 8)                              // k, need
         + ns * kQKI * (8 + 8)                       // parent finish, comm time
         + ns * kQKI * 4 + ns * kQKO * 4             // parent index << 5 | device; children
         + ns * 4 * 9 + 64 + 64;                     // node, inb, deg, outb, odeg, mask, act, free, apos
}

// with the pending counts in shared memory (one byte a node)
__host__ __device__ inline size_t seq_small_smem_bytes_pend(int n, int V) {
  return seq_small_smem_bytes(n) + ((static_cast<size_t>(V) + 15) & ~size_t(15));
}

struct QSm {
  int64_t *F, *tail, *res, *cap;  // [32]
  int64_t *k, *need;              // [ns]
  int64_t *pf, *pc;               // [ns * kQKI]
  int32_t *piq;                   // [ns * kQKI]
  int32_t *sco;                   // [ns * kQKO]
  int32_t *node, *inb, *deg, *outb, *odeg, *act, *freel, *apos;
  uint32_t *mask;                 // [ns] live devices of a slot
  int32_t *cnt;                   // [32] exec-order counters
  int32_t *ctl;                   // [4] init: source count
  uint8_t *pend;                  // [V] parents not yet placed (graphs with in-degrees < 256 and
                                  // V <= kQPendV), else null: the job's pending array in HBM
};

__device__ __forceinline__ QSm seq_small_layout(unsigned char *base, int n) {
  const int ns = seq_small_slots(n);
  QSm m;
  int64_t *p64 = reinterpret_cast<int64_t *>(base);
  m.F = p64;
  m.tail = p64 + 32;
  m.res = p64 + 64;
  m.cap = p64 + 96;
  p64 += 128;
  m.k = p64;
  m.need = p64 + ns;
  p64 += 2 * ns;
  m.pf = p64;
  m.pc = p64 + ns * kQKI;
  p64 += 2 * ns * kQKI;
  int32_t *p32 = reinterpret_cast<int32_t *>(p64);
  m.piq = p32;
  p32 += ns * kQKI;
  m.sco = p32;
  p32 += ns * kQKO;
  m.node = p32;
  m.inb = p32 + ns;
  m.deg = p32 + 2 * ns;
  m.outb = p32 + 3 * ns;
  m.odeg = p32 + 4 * ns;
  m.act = p32 + 5 * ns;
  m.freel = p32 + 6 * ns;
  m.apos = p32 + 7 * ns;
  m.mask = reinterpret_cast<uint32_t *>(p32 + 8 * ns);
  p32 += 9 * ns;
  m.cnt = p32;
  m.ctl = p32 + 32;
  m.pend = reinterpret_cast<uint8_t *>(p32 + 48);
  return m;
}

// Parent k of a ready slot: (index << 5 | device, finish, comm time).
struct QPar {
  int iq;
  int64_t f, c;
};

__device__ __forceinline__ QPar seq_parent(const QSm &m, const DJob &jb, const DGraph &g, const DPrep &pr, int s,
                                           int k) {
  QPar r;
  if (k < kQKI) {
    r.iq = m.piq[s * kQKI + k];
    r.f = m.pf[s * kQKI + k];
    r.c = m.pc[s * kQKI + k];
  } else {
    const int x = m.inb[s] + k;
    const int i = __ldg(g.in_src + x);
    r.iq = i << 5 | jb.device_of[i];
    r.f = jb.finish[i];
    r.c = __ldg(pr.in_c + x);
  }
  return r;
}

// schedulable_time(j, q) of ready slot s on the live tails (placers.cpp:43-79).
// Branch-free per parent (lanes of a warp hold pairs whose parents take
// different cases: local, cached, a new transfer), so the warp issues each
// parent's step once instead of once per case.
// The fold's new transfers (uncached remote parents, in order) are its commit
// recipe: nt of them, the first two as (parent << 5 | device, arrival).
struct QRecipe {
  int nt, a0, a1;
  int64_t t0, t1;
};

__device__ __forceinline__ int64_t seq_key(const QSm &m, const DJob &jb, const DGraph &g, const DPrep &pr,
                                           const int64_t *__restrict__ cache, int n, int s, int q, QRecipe &rc) {
  rc.nt = 0;
  int64_t key = m.F[q];
  int64_t T = m.tail[q];
  const int deg = m.deg[s];
  const int kk = deg < kQKI ? deg : kQKI;
  const int base = s * kQKI;
  for (int k = 0; k < kk; ++k) {
    const int iq = m.piq[base + k];
    const int64_t f = m.pf[base + k], c = m.pc[base + k];
    const int qi = iq & 31;
    const bool local = qi == q;
    // (a local parent reads its own row: a harmless valid address)
    const int64_t ca = cache[(iq >> 5) * n + q];
    const bool cached = !local && ca >= 0;
    const int64_t tn = max64(max64(f, T), m.tail[qi]) + c;
    const int64_t term = local ? f : (cached ? max64(f, ca) : tn);
    const bool xfer = !local && !cached;
    T = xfer ? tn : T;
    key = max64(key, term);
    if (xfer) {
      if (rc.nt == 0) {
        rc.a0 = iq;
        rc.t0 = tn;
      } else if (rc.nt == 1) {
        rc.a1 = iq;
        rc.t1 = tn;
      }
      ++rc.nt;
    }
  }
  for (int k = kQKI; k < deg; ++k) {  // parents past the slot record: from the graph
    const QPar a = seq_parent(m, jb, g, pr, s, k);
    const int qi = a.iq & 31, i = a.iq >> 5;
    if (qi == q) {
      key = max64(key, a.f);
    } else {
      const int64_t ca = cache[static_cast<int64_t>(i) * n + q];
      if (ca >= 0) {
        key = max64(key, max64(a.f, ca));
      } else {
        T = max64(max64(a.f, T), m.tail[qi]) + a.c;
        key = max64(key, T);
        rc.nt += 3;  // (past the slot record: the commit replays the full fold)
      }
    }
  }
  return key;
}

template <bool kProf>
__global__ void __launch_bounds__(32 * kQWarps, 1)
    k_place_seq_small(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs,
                      const DPrep *preps) {
  extern __shared__ __align__(16) unsigned char smem[];
  if (blockIdx.x >= njobs) return;
  const DJob jb = jobs[order[blockIdx.x]];
  if (jb.skip || jb.sdone == nullptr) return;
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // per-phase SM cycles (profiling plans only; lane 0 of the scheduling warp)
  int64_t prof[kProfSlots] = {};
  int64_t prof_last = 0;
  const int64_t prof_t0 = kProf ? clock64() : 0;
#define QMARK(slot)                        \
  if (kProf) {                             \
    const int64_t now_ = clock64();        \
    prof[slot] += now_ - prof_last;        \
    prof_last = now_;                      \
  }
  if (g.flags[0] != g.V || g.flags[1]) {  // the reference's validation order: cycle, then bytes
    if (tid == 0) {
      set_err(jb.err, kValidation, g.flags[0] != g.V ? E_CYCLE : E_NEG_BYTES, 0, 0);
      *jb.sdone = 1;
    }
    return;
  }
  const int V = g.V, n = jb.n;
  if (*pr.cbad || g.flags[2] || n > 32 || n < 1 || V <= 0 || V >= (1 << 26)) return;  // general kernels
  const int ns = seq_small_slots(n);
  QSm m = seq_small_layout(smem, n);
  int64_t *__restrict__ cache = jb.K;  // [V * n] arrival of producer i on device q, -1 none

  // ---- init (whole CTA): per-node state, the sources as the first slots ----
  if (tid == 0) m.ctl[0] = 0;
  if (tid < 32) {
    m.F[tid] = 0;
    m.tail[tid] = 0;
    m.res[tid] = 0;
    m.cap[tid] = tid < n ? jb.cap[tid] : 0;
  }
  __syncthreads();
  const uint32_t full = n >= 32 ? 0xffffffffu : (1u << n) - 1u;
  // pending counts: bytes in shared memory when every in-degree fits one and
  // the slot tables plus V bytes fit the SM (the host sizes the launch alike)
  const bool pend_s = jb.maxin < 256 && V <= kQPendV && seq_small_smem_bytes_pend(n, V) <= kQSmemMax;
  for (int j = tid; j < V; j += 32 * kQWarps) {
    const int ib = g.in_off[j], indeg = g.in_off[j + 1] - ib;
    if (pend_s)
      m.pend[j] = static_cast<uint8_t>(indeg);
    else
      jb.pending[j] = indeg;
    jb.device_of[j] = -1;
    if (indeg == 0) {
      const int s = atomicAdd(m.ctl, 1);
      if (s < ns) {
        const int ob = g.out_off[j], od = g.out_off[j + 1] - ob;
        m.node[s] = j;
        m.k[s] = g.k[j];
        m.need[s] = g.need[j];
        m.inb[s] = ib;
        m.deg[s] = 0;
        m.outb[s] = ob;
        m.odeg[s] = od;
        for (int k = 0; k < od && k < kQKO; ++k) m.sco[s * kQKO + k] = g.edst[ob + k];
        m.mask[s] = full;
        m.act[s] = s;
        m.apos[s] = s;
      }
    }
  }
  __syncthreads();
  if (warp != 0) return;
  int R = m.ctl[0];
  if (R * n > kQPairs) return;  // frontier too wide from the start
  for (int s = R + lane; s < ns; s += 32) m.freel[s - R] = s;  // free slots, popped from the end
  int nfree = ns - R;
  // pair x = lane + 32 t <-> (active position a, device q): stepped, no division
  const int a0 = lane / n, q0 = lane - (lane / n) * n, da = 32 / n, dq = 32 - (32 / n) * n;
  __syncwarp();

  int placed = 0, nexcl = 0, minptr = 0;
  uint32_t exclm = 0;
  int64_t discarded = 0, excluded = 0;
  int err_status = 0, err_code = 0, err_node = 0;
  bool overflow = false;

  if (kProf) prof_last = clock64();
  while (placed < V) {
    if (kProf) ++prof[P_STEPS];
    // ---- keys + selection ---------------------------------------------------
    const int np = R * n;
    int64_t bt = kInf;
    unsigned bi = 0xffffffffu;
    int bs = -1;
    QRecipe best;
    best.nt = 0;
    for (int x = lane, a = a0, q = q0; x < np; x += 32, a += da, q += dq) {
      if (q >= n) {
        q -= n;
        ++a;
      }
      const int s = m.act[a];
      if (!((m.mask[s] >> q) & 1u)) continue;
      QRecipe rc;
      const int64_t key = seq_key(m, jb, g, pr, cache, n, s, q, rc);
      const unsigned id = static_cast<unsigned>(m.node[s]) << 5 | static_cast<unsigned>(q);
      if (key < bt || (key == bt && id < bi)) {
        bt = key;
        bi = id;
        bs = s;
        best = rc;
      }
    }
    const int64_t mykey = bt;
    const unsigned myid = bi;
    warp_argmin_u(bt, bi);
    if (bi == 0xffffffffu) {
      err_status = kInfeasible;
      err_code = E_NO_PAIR;
      break;
    }
    const unsigned owner = __ballot_sync(kFull, mykey == bt && myid == bi);
    const int olane = __ffs(owner) - 1;
    const int s = __shfl_sync(kFull, bs, olane);
    const int nt = __shfl_sync(kFull, best.nt, olane);
    const int j = static_cast<int>(bi >> 5), p = static_cast<int>(bi & 31u);
    const int64_t t = bt;
    const int64_t needj = m.need[s];
    QMARK(P_ARGMIN);

    if (m.res[p] + needj > m.cap[p]) {
      // ---- discard (placers.cpp:203-219) ------------------------------------
      const uint32_t left = m.mask[s] & ~(1u << p);
      __syncwarp();
      if (lane == 0) m.mask[s] = left;
      if (left == 0) {
        err_status = kInfeasible;
        err_code = E_FITS_NONE;
        err_node = j;
        break;
      }
      ++discarded;
      // smallest need among the unplaced nodes (the `remaining` multiset)
      int64_t minrem = 0;
      if (lane == 0) {
        while (jb.device_of[g.need_order[minptr]] >= 0) ++minptr;
        minrem = g.need[g.need_order[minptr]];
      }
      minrem = __shfl_sync(kFull, minrem, 0);
      if (m.res[p] + minrem > m.cap[p]) {
        // exclusion: every unplaced (j2, p) dies, ascending j2; unready nodes
        // carry no discards, so they die together when the last device goes
        ++excluded;
        ++nexcl;
        exclm |= 1u << p;
        __syncwarp();
        int first_dead = INT32_MAX;
        for (int a = lane; a < R; a += 32) {
          const int s2 = m.act[a];
          const uint32_t mk = m.mask[s2];
          if ((mk >> p) & 1u) {
            m.mask[s2] = mk & ~(1u << p);
            if ((mk & ~(1u << p)) == 0) first_dead = min(first_dead, m.node[s2]);
          }
        }
        if (nexcl == n)
          for (int x = lane; x < V; x += 32)
            if (jb.device_of[x] < 0) first_dead = min(first_dead, x);
        first_dead = warp_min_i32(first_dead);
        if (first_dead != INT32_MAX) {
          err_status = kInfeasible;
          err_code = E_FITS_NONE;
          err_node = first_dead;
          break;
        }
      }
      __syncwarp();
      QMARK(P_DISCARD);
      continue;
    }

    // ---- commit (placers.cpp:221-233) -----------------------------------------
    const int64_t fin = t + m.k[s];
    const int deg = m.deg[s];
    // the children first: their pending-count atomics are in flight while
    // lane 0 folds the transfers
    const int od = m.odeg[s];
    int child = -1;
    bool ready = false;
    if (!pend_s && lane < od && lane < kQKO) {
      child = m.sco[s * kQKO + lane];
      ready = atomicSub(jb.pending + child, 1) == 1;
    }
    if (lane < n) cache[static_cast<int64_t>(j) * n + lane] = -1;  // j's arrival row
    if (nt <= 2) {
      // commit_schedulable_time from the winner's recipe: its fold ran on
      // this very state, so the commit is the recipe's stores
      if (lane == olane && nt > 0) {
        m.tail[best.a0 & 31] = best.t0;
        cache[(best.a0 >> 5) * n + p] = best.t0;
        if (nt > 1) {
          m.tail[best.a1 & 31] = best.t1;
          cache[(best.a1 >> 5) * n + p] = best.t1;
        }
        m.tail[p] = nt > 1 ? best.t1 : best.t0;
      }
    } else if (lane == 0) {
      int64_t Tp = m.tail[p];
      for (int k = 0; k < deg; ++k) {
        const QPar a = seq_parent(m, jb, g, pr, s, k);
        const int qi = a.iq & 31, i = a.iq >> 5;
        if (qi == p) continue;
        int64_t *slot = cache + static_cast<int64_t>(i) * n + p;
        if (*slot >= 0) continue;
        const int64_t term = max64(a.f, max64(m.tail[qi], Tp)) + a.c;
        m.tail[qi] = term;
        Tp = term;
        *slot = term;
      }
      m.tail[p] = Tp;
    }
    if (lane == 0) {
      m.F[p] = fin;
      m.res[p] += needj;
      jb.device_of[j] = p;
      jb.start[j] = t;
      jb.finish[j] = fin;
      jb.cseq[placed] = j;
      // the committed slot leaves: the last active slot takes its place
      const int pos = m.apos[s];
      const int last = m.act[R - 1];
      m.act[pos] = last;
      m.apos[last] = pos;
    }
    ++placed;
    --R;
    if (kProf) ++prof[P_COMMITS];
    QMARK(P_COMMIT);
    __syncwarp();  // lane 0's finish / device and slot moves before the children read them

    // ---- readiness of the children (placers.cpp:256-268) -----------------------
    for (int y0 = 0; y0 < od; y0 += 32) {
      // (HBM counts: the slot's first kQKO children were decremented above)
      const int y = y0 + lane;
      const bool fresh = pend_s || y0 > 0 || lane >= kQKO;
      if (fresh) {
        child = -1;
        ready = false;
        if (y < od) child = y < kQKO ? m.sco[s * kQKO + y] : __ldg(g.edst + m.outb[s] + y);
      }
      if (pend_s) {
        // one warp owns the counts, and a node's children are distinct (meta
        // edges are unique, checked when the graph is made)
        if (child >= 0) {
          const int v = static_cast<int>(m.pend[child]) - 1;
          m.pend[child] = static_cast<uint8_t>(v);
          ready = v == 0;
        }
      } else if (fresh && child >= 0) {
        ready = atomicSub(jb.pending + child, 1) == 1;
      }
      const unsigned b = __ballot_sync(kFull, ready);
      const int nn = __popc(b);
      if (nn == 0) continue;
      if ((R + nn) * n > kQPairs || nn > nfree) {
        overflow = true;
        break;
      }
      if (ready) {
        const int r = __popc(b & ((1u << lane) - 1u));
        const int s2 = m.freel[nfree - 1 - r];
        const int ib = __ldg(g.in_off + child), ob = __ldg(g.out_off + child);
        const int ie = __ldg(g.in_off + child + 1), oe = __ldg(g.out_off + child + 1);
        m.act[R + r] = s2;
        m.apos[s2] = R + r;
        m.node[s2] = child;
        m.k[s2] = __ldg(g.k + child);
        m.need[s2] = __ldg(g.need + child);
        m.inb[s2] = ib;
        m.deg[s2] = ie - ib;
        m.outb[s2] = ob;
        m.odeg[s2] = oe - ob;
        m.mask[s2] = full & ~exclm;
      }
      __syncwarp();
      QMARK(P_READY);
      // the new slots' records: lanes over (new slot, k < 8) parents and children
      for (int it = lane; it < nn * kQKI; it += 32) {
        const int r = it / kQKI, k = it - r * kQKI;
        const int s3 = m.act[R + r];
        if (k < m.deg[s3]) {
          const uint2 ip = __ldg(pr.in_pack + m.inb[s3] + k);
          const int i = static_cast<int>(ip.x);
          // the node just committed: from registers (its stores may still be
          // on their way to L2)
          m.piq[s3 * kQKI + k] = i << 5 | (i == j ? p : jb.device_of[i]);
          m.pf[s3 * kQKI + k] = i == j ? fin : jb.finish[i];
          m.pc[s3 * kQKI + k] = static_cast<int64_t>(ip.y & 0xffffu);
        }
        if (k < m.odeg[s3]) m.sco[s3 * kQKO + k] = __ldg(g.edst + m.outb[s3] + k);
      }
      R += nn;
      nfree -= nn;
      __syncwarp();
      QMARK(P_ROWS);
    }
    if (overflow) break;
    if (lane == 0) m.freel[nfree] = s;  // the committed slot is free once its children are read
    ++nfree;
    __syncwarp();
  }
#undef QMARK

  if (overflow) return;  // the general kernel places it
  if (err_status) {
    if (lane == 0) {
      set_err(jb.err, err_status, err_code, err_node, 0);
      *jb.sdone = 1;
    }
    return;
  }
  __threadfence_block();
  __syncwarp();
  Ctx c;
  c.V = V;
  c.n = n;
  c.device_of = jb.device_of;
  c.start = jb.start;
  c.cseq = jb.cseq;
  emit_exec_order(c, jb, m.cnt, lane);
  if (lane == 0) {
    jb.stats[0] = discarded;
    jb.stats[1] = excluded;
    jb.stats[2] = 0;
    set_err(jb.err, kOk, E_NONE, 0, 0);
    *jb.sdone = 1;
    if (kProf && jb.prof) {
      prof[P_TOTAL] = clock64() - prof_t0;
      for (int k = 0; k < kProfSlots; ++k) jb.prof[k] = prof[k];
    }
  }
}

// launch bytes for a job: the slot tables, plus its pending counts when they fit
size_t seq_small_smem_bytes_host(int n, int V, int maxin) {
  const size_t b = seq_small_smem_bytes_pend(n, V);
  return maxin < 256 && V <= kQPendV && b <= kQSmemMax ? b : seq_small_smem_bytes(n);
}

// One CTA per job (`order` lists the K2q jobs).
void launch_seq_small(const DJob *jobs, const int32_t *order, int nj, const DGraph *graphs, const DPrep *preps,
                      size_t smem, bool prof, cudaStream_t s) {
  if (nj <= 0) return;
  auto kern = prof ? k_place_seq_small<true> : k_place_seq_small<false>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  kern<<<nj, 32 * kQWarps, smem, s>>>(jobs, order, nj, graphs, preps);
}

}  // namespace bx

// K2s — the small-frontier list placer (parallel comm mode, m-ETF / m-SCT).
//
// Same contract as K2 (place_list, proj/src/placers.cpp:115-295, in its
// exact-argmin form): every step takes the lexicographic minimum of
// (key(j,p), j, p) over the live pairs and commits or discards it.
//
// Model-shaped training graphs keep a tiny ready frontier under list
// scheduling (Inception/GNMT/Transformer meta graphs and the reference's
// layered-chain family: 3-6 ready nodes on average), so a placement is a
// chain of V dependent steps over a few dozen pairs. This kernel is built
// for that chain: ONE warp per problem, no CTA barriers, every mutable
// per-node value in shared memory, and every live pair held in a register
// of some lane (R*n <= 256, at most 8 pairs per lane).
//
// A round:
//   1. keys: each lane forms key = max(dev_free[q], DR[s][q]) (+ the m-SCT
//      awake floor, placers.cpp:147-156) for its pairs from shared memory,
//      as one 64-bit word (key << 32 | node << 5 | q) — (key, node, device)
//      order in a single unsigned compare;
//   2. selection: a two-REDUX warp minimum gives the global argmin; a pair
//      that does not fit is discarded on the spot (placers.cpp:203-219);
//      a pair that fits commits. After committing (j, p) at t every key that
//      can change or appear is >= t + k_j (column p's keys are >= the new
//      dev_free[p]; a newly cached parent only touches column p; a newly
//      ready child has j as a parent), so the next minimum among the
//      untouched pairs commits in the same round while its key is below the
//      least such finish time T. m-SCT: a lifted reservation may lower the
//      keys of its column, which then drops out of the round and lowers T to
//      its dev_free (every key of a column is >= its dev_free);
//   3. one batched update for all of the round's commits: cache arrivals
//      (commit_schedulable_time, :95-101), readiness (:256-268), new
//      data-ready rows and the re-keys of consumers whose parent tensor just
//      landed (:271-279).
//
// Data-ready time DR[s][q] = max over parents i of: finish_i (same device),
// max(finish_i, cache[i][q]) (tensor already on q), finish_i + c_e otherwise
// (placers.cpp:55-61). In parallel mode the cache holds finish_i + c of the
// edge whose consumer first landed on q, so for a producer whose out-edges
// all carry the same comm time the cache never changes a term: only the
// remaining ("non-uniform") producers get cache rows (nu index x n, shared
// memory), each entry the 16-bit comm time of the edge that brought the
// tensor (its arrival is the producer's finish plus that).
//
// Times are int32 here: the kernel first checks sum(k) + (V + 2) * c_max
// < 2^31 (every start is at most the previous largest finish + c_max, also
// for the m-SCT floor), 0 <= c < 2^16 - 1 and in-degrees below 2^16 - 1
// (16-bit pending counters). Any check that fails — or a frontier beyond
// 256 pairs at any point — leaves sdone = 0 and the general kernels
// (listsched.cu), launched behind this one, place the job instead.
//
// Per-node state is 12 bytes of shared memory (finish/device, pending,
// ready slot), so graphs up to ~12k meta nodes fit; the rest of the SM's
// 256 KB goes to L1, which three helper warps fill with the graph arrays
// before the scheduling warp needs them.
#include "sched_common.cuh"

namespace bx {

constexpr int kSP = 8;                  // pairs per lane
constexpr int kSPairs = 32 * kSP;       // R * n <= 256
constexpr int kSCommits = 32;           // commits per round
constexpr int32_t kSDead = 0x7fffffff;  // DR of a discarded / excluded pair
constexpr uint64_t kSNone = ~0ull;

__device__ __forceinline__ uint64_t sm_min_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_min_sync(kFull, hi);
  const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}

__device__ __forceinline__ int sm_dev(uint64_t info) { return static_cast<int>(static_cast<uint32_t>(info)); }
__device__ __forceinline__ int32_t sm_fin(uint64_t info) { return static_cast<int32_t>(info >> 32); }

// Shared-memory layout of one problem (host: small_smem_bytes).
struct SSm {
  int32_t *F, *awf, *awu, *excl;  // [32] per device
  int64_t *res, *cap;             // [32]
  uint64_t *info;                 // [V] finish << 32 | device (0xffffffff: unplaced)
  uint16_t *pending;              // [V] parents not yet placed (decremented as 32-bit words)
  int16_t *rpos;                  // [V] ready slot of a node, -1 none
  uint16_t *nuc;                  // [nucap * n] per non-uniform producer and device: comm time of the
                                  // edge that first brought its tensor there (arrival = finish + it), 0xffff absent
  // ready slots
  int32_t *node, *kk, *inb, *ine, *outb, *oute, *alive, *urg;  // [kSPairs]
  int64_t *need;                                               // [kSPairs]
  int32_t *dr;                                                 // [kSPairs]  DR[s * n + q]
  // per round
  int32_t *cj, *cp, *cfin, *cs, *pin, *pout, *ord;  // [kSCommits + 1]
  int32_t *nci, *ncp;                               // [nccap] newly cached (producer, device)
  int32_t *newn;                                    // [kSPairs] newly ready nodes
  int32_t *scal;                                    // [32] exec-order counters
};

__host__ __device__ inline size_t small_smem_bytes(int V, int n, int nucap, int nccap) {
  (void)n;
  size_t b = 0;
  b += 4 * 32 * 4 + 2 * 32 * 8;
  b += size_t(V) * 8 + 2 * ((size_t(V) * 2 + 3) & ~size_t(3));
  b += (size_t(nucap) * n * 2 + 7) & ~size_t(7);
  b += kSPairs * (8 * 4 + 8 + 4);
  b += 7 * (kSCommits + 1) * 4 + 4;
  b += 2 * size_t(nccap) * 4 + kSPairs * 4 + 32 * 4;
  return b + 64;
}

__device__ __forceinline__ SSm small_layout(unsigned char *base, int V, int n, int nucap, int nccap) {
  SSm m;
  int64_t *p64 = reinterpret_cast<int64_t *>(base);
  m.res = p64;
  m.cap = p64 + 32;
  m.info = reinterpret_cast<uint64_t *>(p64 + 64);
  m.need = reinterpret_cast<int64_t *>(m.info + V);
  int32_t *p32 = reinterpret_cast<int32_t *>(m.need + kSPairs);
  m.F = p32;
  m.awf = p32 + 32;
  m.awu = p32 + 64;
  m.excl = p32 + 96;
  p32 += 128;
  const int vw = (V + 1) / 2;  // int32 words of a [V] 16-bit array
  m.pending = reinterpret_cast<uint16_t *>(p32);
  m.rpos = reinterpret_cast<int16_t *>(p32 + vw);
  p32 += 2 * vw;
  m.nuc = reinterpret_cast<uint16_t *>(p32);
  p32 += (nucap * n + 1) / 2;
  m.node = p32;
  m.kk = p32 + kSPairs;
  m.inb = p32 + 2 * kSPairs;
  m.ine = p32 + 3 * kSPairs;
  m.outb = p32 + 4 * kSPairs;
  m.oute = p32 + 5 * kSPairs;
  m.alive = p32 + 6 * kSPairs;
  m.urg = p32 + 7 * kSPairs;
  m.dr = p32 + 8 * kSPairs;
  p32 += 9 * kSPairs;
  constexpr int C1 = kSCommits + 1;
  m.cj = p32;
  m.cp = p32 + C1;
  m.cfin = p32 + 2 * C1;
  m.cs = p32 + 3 * C1;
  m.pin = p32 + 4 * C1;
  m.pout = p32 + 5 * C1;
  m.ord = p32 + 6 * C1;
  p32 += 7 * C1;
  m.nci = p32;
  m.ncp = p32 + nccap;
  m.newn = p32 + 2 * nccap;
  m.scal = m.newn + kSPairs;
  return m;
}

// Read-only graph view (global memory, read through the non-coherent path).
struct SGraph {
  const int32_t *__restrict__ in_off, *__restrict__ in_src, *__restrict__ out_off, *__restrict__ out_dst;
  const int32_t *__restrict__ c32, *__restrict__ nu, *__restrict__ fav;
  const int64_t *__restrict__ k, *__restrict__ need;
  const int32_t *__restrict__ need_order;
};

// DR of node c on device q (and, for m-SCT, its urgency: max over parents of
// finish + c_e ignoring caches, placers.cpp:259-266).
template <bool kUrg>
__device__ __forceinline__ int32_t small_dr(const SSm &m, const SGraph &G, int n, int lo, int hi, int q,
                                            int32_t &urg) {
  int32_t t = 0, u = 0;
  int x = lo;
  for (; x + 1 < hi; x += 2) {
    const int i0 = __ldg(G.in_src + x), i1 = __ldg(G.in_src + x + 1);
    const int32_t c0 = __ldg(G.c32 + x), c1 = __ldg(G.c32 + x + 1);
    const int u0 = __ldg(G.nu + i0), u1 = __ldg(G.nu + i1);
    const uint64_t a0 = m.info[i0], a1 = m.info[i1];
    const int32_t f0 = sm_fin(a0), f1 = sm_fin(a1);
    int32_t t0, t1;
    if (sm_dev(a0) == q) {
      t0 = f0;
    } else {
      const unsigned z = u0 >= 0 ? m.nuc[u0 * n + q] : 0xffffu;
      t0 = f0 + (z != 0xffffu ? static_cast<int32_t>(z) : c0);
    }
    if (sm_dev(a1) == q) {
      t1 = f1;
    } else {
      const unsigned z = u1 >= 0 ? m.nuc[u1 * n + q] : 0xffffu;
      t1 = f1 + (z != 0xffffu ? static_cast<int32_t>(z) : c1);
    }
    t = max(t, max(t0, t1));
    if (kUrg) u = max(u, max(f0 + c0, f1 + c1));
  }
  if (x < hi) {
    const int i0 = __ldg(G.in_src + x);
    const int32_t c0 = __ldg(G.c32 + x);
    const int u0 = __ldg(G.nu + i0);
    const uint64_t a0 = m.info[i0];
    const int32_t f0 = sm_fin(a0);
    int32_t t0;
    if (sm_dev(a0) == q) {
      t0 = f0;
    } else {
      const unsigned z = u0 >= 0 ? m.nuc[u0 * n + q] : 0xffffu;
      t0 = f0 + (z != 0xffffu ? static_cast<int32_t>(z) : c0);
    }
    t = max(t, t0);
    if (kUrg) u = max(u, f0 + c0);
  }
  urg = u;
  return t;
}

// Fills slot fields for newly ready nodes in slots [R0, R0 + cnt) (node ids
// already in m.node).
__device__ __forceinline__ void small_fill_slots(const SSm &m, const SGraph &G, int R0, int cnt, int alive,
                                                 int lane) {
  for (int x = lane; x < cnt; x += 32) {
    const int s = R0 + x, c = m.node[s];
    m.rpos[c] = s;
    m.need[s] = __ldg(G.need + c);
    m.kk[s] = static_cast<int32_t>(__ldg(G.k + c));
    m.inb[s] = __ldg(G.in_off + c);
    m.ine[s] = __ldg(G.in_off + c + 1);
    m.outb[s] = __ldg(G.out_off + c);
    m.oute[s] = __ldg(G.out_off + c + 1);
    m.alive[s] = alive;
    m.urg[s] = 0;
  }
}

// Per-problem loop state kept in registers (identical in every lane).
struct SRun {
  int R, placed, nexcl, minptr;
  int64_t discarded, excluded, awake;
  int err_status, err_code, err_node;
  int32_t cmax;
  int V, n, d32, r32, s0, q0;
};

// Steps 1-2 of a round with P pairs per lane (R * n <= 32 P): keys, then
// exact commits / discards below the threshold. Commits land in m.cj/cp/
// cfin/cs; returns their count (sin/sout: their total in/out-degree),
// `progress` false when no live pair exists at all.
template <int P, bool kSct>
__device__ __forceinline__ int small_select(const SSm &m, const SGraph &G, const DJob &jb, SRun &st, int nccap,
                                            int lane, int &sin, int &sout, bool &progress) {
  const int n = st.n;
  const int np = st.R * n;
  uint64_t ck[P];
  int32_t kq[P];  // k of the pair's node
  int32_t sq[P];  // slot << 5 | device
  unsigned fitm = 0;
  {
    int s = st.s0, q = st.q0;
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int x = lane + 32 * u;
      ck[u] = kSNone;
      kq[u] = 0;
      sq[u] = s << 5 | q;
      if (x < np) {
        const int32_t d = m.dr[x];
        if (d != kSDead && !m.excl[q]) {
          const int node = m.node[s];
          int32_t key = max(m.F[q], d);
          if (kSct) {
            const int a = m.awf[q];
            if (a >= 0 && a != node) key = max(key, min(m.awu[q], m.urg[s]));
          }
          ck[u] = (static_cast<uint64_t>(static_cast<uint32_t>(key)) << 32) |
                  (static_cast<uint32_t>(node) << 5 | static_cast<uint32_t>(q));
          kq[u] = m.kk[s];
          if (m.res[q] + m.need[s] <= m.cap[q]) fitm |= 1u << u;
        }
      }
      if (P > 1) {
        s += st.d32;
        q += st.r32;
        if (q >= n) {
          q -= n;
          ++s;
        }
      }
    }
  }
  uint32_t T = 0xffffffffu;
  int nc = 0;
  sin = sout = 0;
  progress = false;
  while (true) {
    uint64_t best = ck[0];
#pragma unroll
    for (int u = 1; u < P; ++u) best = ck[u] < best ? ck[u] : best;
    const uint64_t w = sm_min_u64(best);
    if (w >= (static_cast<uint64_t>(T) << 32)) break;
    const bool own = best == w;
    const int ol = __ffs(__ballot_sync(kFull, own)) - 1;
    int msq = 0, mk = 0;
    if (own) {
#pragma unroll
      for (int u = 0; u < P; ++u)
        if (ck[u] == w) {
          msq = sq[u] | (((fitm >> u) & 1) << 30);
          mk = kq[u];
          ck[u] = kSNone;
        }
    }
    msq = __shfl_sync(kFull, msq, ol);
    mk = __shfl_sync(kFull, mk, ol);
    const int32_t t = static_cast<int32_t>(w >> 32);
    const int j = static_cast<int>((static_cast<uint32_t>(w)) >> 5);
    const int p = static_cast<int>(w & 31u);
    const int s = (msq >> 5) & 0x1ffffff;
    progress = true;
    if (!(msq >> 30)) {
      // ---- discard (placers.cpp:203-219) ----
      int left = 0;
      if (lane == 0) {
        m.dr[s * n + p] = kSDead;
        left = --m.alive[s];
      }
      left = __shfl_sync(kFull, left, 0);
      __syncwarp();
      if (left == 0) {
        st.err_status = kInfeasible;
        st.err_code = E_FITS_NONE;
        st.err_node = j;
        return nc;
      }
      ++st.discarded;
      // smallest need among all unplaced nodes (the `remaining` multiset)
      int64_t minrem = 0;
      if (lane == 0) {
        while (sm_dev(m.info[__ldg(G.need_order + st.minptr)]) >= 0) ++st.minptr;
        minrem = __ldg(G.need + __ldg(G.need_order + st.minptr));
      }
      minrem = __shfl_sync(kFull, minrem, 0);
      if (m.res[p] + minrem > m.cap[p]) {
        // exclusion: every unplaced (j2, p) dies (ascending j2 in the
        // reference; the first node left with no device is the smallest)
        ++st.excluded;
        ++st.nexcl;
        int first_dead = INT32_MAX;
        for (int s2 = lane; s2 < st.R; s2 += 32) {
          const int node2 = m.node[s2];
          if (sm_dev(m.info[node2]) >= 0) continue;  // committed earlier this round
          const int x2 = s2 * n + p;
          if (m.dr[x2] != kSDead) {
            m.dr[x2] = kSDead;
            if (--m.alive[s2] == 0) first_dead = min(first_dead, node2);
          }
        }
        if (st.nexcl == n)
          for (int x = lane; x < st.V; x += 32)
            if (sm_dev(m.info[x]) < 0) first_dead = min(first_dead, x);
        first_dead = static_cast<int>(__reduce_min_sync(kFull, static_cast<unsigned>(first_dead)));
        if (first_dead != INT32_MAX) {
          st.err_status = kInfeasible;
          st.err_code = E_FITS_NONE;
          st.err_node = first_dead;
          return nc;
        }
        if (lane == 0) m.excl[p] = 1;
#pragma unroll
        for (int u = 0; u < P; ++u)
          if ((sq[u] & 31) == p) ck[u] = kSNone;
      }
      __syncwarp();
      continue;
    }
    // ---- commit (placers.cpp:221-233) ----
    const int32_t fin = t + mk;
    if (lane == 0) {
      m.cj[nc] = j;
      m.cp[nc] = p;
      m.cfin[nc] = fin;
      m.cs[nc] = s;
      m.F[p] = fin;
      m.res[p] += m.need[s];
      m.info[j] = (static_cast<uint64_t>(static_cast<uint32_t>(fin)) << 32) | static_cast<uint32_t>(p);
      jb.device_of[j] = p;
      jb.start[j] = t;
      jb.cseq[st.placed] = j;
    }
    ++st.placed;
    ++nc;
    T = min(T, static_cast<uint32_t>(fin));
#pragma unroll
    for (int u = 0; u < P; ++u)
      if ((sq[u] & 31) == p || (static_cast<uint32_t>(ck[u]) >> 5) == static_cast<uint32_t>(j)) ck[u] = kSNone;
    if (kSct) {
      // awake reservations (placers.cpp:235-254): columns whose reservation
      // awaited j are lifted — their keys may drop, so they leave the round
      // and bound it by their dev_free
      const bool lifted = lane < n && lane != p && m.awf[lane] == j;
      const unsigned lm = __ballot_sync(kFull, lifted);
      uint32_t fq = 0xffffffffu;
      if (lifted) {
        m.awf[lane] = -1;
        fq = static_cast<uint32_t>(m.F[lane]);
      }
      T = min(T, __reduce_min_sync(kFull, fq));
#pragma unroll
      for (int u = 0; u < P; ++u)
        if ((lm >> (sq[u] & 31)) & 1) ck[u] = kSNone;
      int got = 0;
      if (lane == 0) {
        m.awf[p] = -1;
        const int h = __ldg(G.fav + j);
        if (h >= 0 && sm_dev(m.info[h]) < 0) {
          m.awf[p] = h;
          m.awu[p] = fin + st.cmax;
          got = 1;
        }
      }
      st.awake += __shfl_sync(kFull, got, 0);
    }
    sin += m.ine[s] - m.inb[s];
    sout += m.oute[s] - m.outb[s];
    __syncwarp();
    if (nc == kSCommits || sin + jb.maxin > nccap || st.placed == st.V) break;
  }
  return nc;
}

// Brings [p, p + bytes) into this SM's L1 (one 16-byte load per 32-byte
// sector, results folded into a value the caller keeps alive).
__device__ __forceinline__ unsigned warm_l1(const void *p, size_t bytes, int tid, int nthreads) {
  const char *b = static_cast<const char *>(p);
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(b) & ~uintptr_t(31);
  const uintptr_t a1 = reinterpret_cast<uintptr_t>(b + bytes);
  unsigned acc = 0;
  for (uintptr_t a = a0 + 32 * static_cast<uintptr_t>(tid); a < a1; a += 32 * static_cast<uintptr_t>(nthreads)) {
    const uint4 v = __ldg(reinterpret_cast<const uint4 *>(a));
    acc ^= v.x;
  }
  return acc;
}

// One CTA per job: warp 0 schedules; warps 1..kSWarm-1 first pull the
// graph arrays the scheduler reads into the SM's L1 (every one of them is
// read through __ldg, and each scheduling round is a chain of dependent
// loads, so L1 instead of L2 latency on each level), then exit.
constexpr int kSWarm = 4;

template <bool kSct, bool kProf>
__global__ void __launch_bounds__(32 * kSWarm, 1)
    k_place_small(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31;
  if (blockIdx.x >= njobs) return;
  const DJob jb = jobs[order[blockIdx.x]];
  if (jb.skip || jb.sdone == nullptr) return;
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  if (threadIdx.x >= 32) {
    const int tid = threadIdx.x - 32, nt = 32 * (kSWarm - 1);
    const size_t V = static_cast<size_t>(g.V), E = static_cast<size_t>(g.E);
    unsigned acc = warm_l1(g.in_off, 4 * (V + 1), tid, nt) ^ warm_l1(g.out_off, 4 * (V + 1), tid, nt);
    acc ^= warm_l1(g.in_src, 4 * E, tid, nt) ^ warm_l1(pr.in_c32, 4 * E, tid, nt);
    acc ^= warm_l1(pr.nu, 4 * V, tid, nt) ^ warm_l1(g.edst, 4 * E, tid, nt);
    acc ^= warm_l1(g.k, 8 * V, tid, nt) ^ warm_l1(g.need, 8 * V, tid, nt);
    acc ^= warm_l1(g.need_order, 4 * V, tid, nt);
    if (kSct && jb.fav) acc ^= warm_l1(jb.fav, 4 * V, tid, nt);
    asm volatile("" ::"r"(acc));  // keeps the loads
    return;
  }
  if (g.flags[0] != g.V || g.flags[1]) {  // the reference's validation order: cycle, then bytes
    if (lane == 0) {
      set_err(jb.err, kValidation, g.flags[0] != g.V ? E_CYCLE : E_NEG_BYTES, 0, 0);
      *jb.sdone = 1;
    }
    return;
  }
  const int V = g.V, n = jb.n;
  const int64_t cmax64 = *pr.cmax;
  const int nccap = jb.maxin > 1024 ? jb.maxin : 1024;
  // dynamic eligibility (see the header); otherwise the general kernel runs it
  if (*pr.cbad || g.flags[2] || *g.ksum < 0 || *pr.nu_count > jb.nucap || n > 32 || V >= (1 << 26) ||
      cmax64 >= 0xffff || jb.maxin >= 0xffff || *g.ksum + (int64_t(V) + 2) * cmax64 >= int64_t(INT32_MAX))
    return;
  const int32_t cmax = static_cast<int32_t>(cmax64);
  const SSm m = small_layout(smem, V, n, jb.nucap, nccap);
  SGraph G;
  G.in_off = g.in_off;
  G.in_src = g.in_src;
  G.out_off = g.out_off;
  G.out_dst = g.edst;
  G.c32 = pr.in_c32;
  G.nu = pr.nu;
  G.fav = jb.fav;
  G.k = g.k;
  G.need = g.need;
  G.need_order = g.need_order;

  // ---- init ------------------------------------------------------------------
  {
    m.F[lane] = 0;
    m.awf[lane] = -1;
    m.awu[lane] = 0;
    m.excl[lane] = 0;
    m.res[lane] = 0;
    m.cap[lane] = lane < n ? jb.cap[lane] : 0;
    for (int x = lane; x < jb.nucap * n; x += 32) m.nuc[x] = 0xffffu;
  }
  int R = 0;
  bool overflow = false;
  for (int base = 0; base < V; base += 32) {
    const int j = base + lane;
    bool src = false;
    if (j < V) {
      const int indeg = __ldg(G.in_off + j + 1) - __ldg(G.in_off + j);
      m.info[j] = 0xffffffffull;
      m.pending[j] = indeg;
      m.rpos[j] = -1;
      src = indeg == 0;
    }
    const unsigned b = __ballot_sync(kFull, src);
    if (src) {
      const int s = R + __popc(b & ((1u << lane) - 1u));
      if (s < kSPairs) m.node[s] = j;
    }
    R += __popc(b);
  }
  if (R * n > kSPairs) return;  // frontier too wide from the start
  __syncwarp();
  small_fill_slots(m, G, 0, R, n, lane);
  for (int x = lane; x < R * n; x += 32) m.dr[x] = 0;
  __syncwarp();

  // per-lane pair walk: x = lane + 32 u -> (slot, device)
  SRun st;
  st.R = R;
  st.V = V;
  st.n = n;
  st.d32 = 32 / n;
  st.r32 = 32 % n;
  st.s0 = lane / n;
  st.q0 = lane % n;
  st.placed = st.nexcl = st.minptr = 0;
  st.discarded = st.excluded = st.awake = 0;
  st.err_status = st.err_code = st.err_node = 0;
  st.cmax = cmax;
  int64_t prof[kProfSlots];
  int64_t prof_last = 0;
  if (kProf) {
#pragma unroll
    for (int k = 0; k < kProfSlots; ++k) prof[k] = 0;
    prof_last = clock64();
  }
  const int64_t prof_t0 = prof_last;
#define SMARK(slot)                   \
  do {                                \
    if (kProf) {                      \
      int64_t now_ = clock64();       \
      prof[slot] += now_ - prof_last; \
      prof_last = now_;               \
    }                                 \
  } while (0)

  while (st.placed < V) {
    // ---- 1-2. keys and the round's exact commits ------------------------------
    int sin = 0, sout = 0;
    bool progress = false;
    const int np = st.R * n;
    const int nc = np <= 32    ? small_select<1, kSct>(m, G, jb, st, nccap, lane, sin, sout, progress)
                   : np <= 64  ? small_select<2, kSct>(m, G, jb, st, nccap, lane, sin, sout, progress)
                   : np <= 128 ? small_select<4, kSct>(m, G, jb, st, nccap, lane, sin, sout, progress)
                               : small_select<8, kSct>(m, G, jb, st, nccap, lane, sin, sout, progress);
    if (kProf) {
      ++prof[P_STEPS];
      prof[P_COMMITS] += nc;
    }
    SMARK(P_ARGMIN);
    if (st.err_status) break;
    if (!progress) {
      st.err_status = kInfeasible;
      st.err_code = E_NO_PAIR;
      break;
    }
    if (nc == 0) continue;

    // ---- 3. batched update of the round's commits ------------------------------
    // per-commit in/out-degree prefixes (a single commit needs none)
    if (nc > 1) {
      int din = 0, dout = 0;
      if (lane < nc) {
        const int s = m.cs[lane];
        din = m.ine[s] - m.inb[s];
        dout = m.oute[s] - m.outb[s];
      }
      int a = din, b = dout;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int a2 = __shfl_up_sync(kFull, a, o), b2 = __shfl_up_sync(kFull, b, o);
        if (lane >= o) {
          a += a2;
          b += b2;
        }
      }
      if (lane < nc) {
        m.pin[lane] = a - din;
        m.pout[lane] = b - dout;
      }
    } else if (lane == 0) {
      m.pin[0] = m.pout[0] = 0;
    }
    __syncwarp();
    // A: cache arrivals of remote non-uniform parents; B: readiness
    int nnc = 0;
    for (int base = 0; base < sin; base += 32) {
      const int idx = base + lane;
      bool fresh = false;
      int i = 0, pr_ = 0;
      if (idx < sin) {
        int r = 0;
        while (r + 1 < nc && m.pin[r + 1] <= idx) ++r;
        const int x = m.inb[m.cs[r]] + idx - m.pin[r];
        pr_ = m.cp[r];
        i = __ldg(G.in_src + x);
        const uint64_t a = m.info[i];
        if (sm_dev(a) != pr_) {
          const int u = __ldg(G.nu + i);
          if (u >= 0) {
            // one commit per device per round, so no two lanes share a slot
            uint16_t *slot = m.nuc + u * n + pr_;
            if (*slot == 0xffffu) {
              *slot = static_cast<uint16_t>(__ldg(G.c32 + x));
              fresh = true;
            }
          }
        }
      }
      const unsigned b = __ballot_sync(kFull, fresh);
      if (fresh) {
        const int at = nnc + __popc(b & ((1u << lane) - 1u));
        m.nci[at] = i;
        m.ncp[at] = pr_;
      }
      nnc += __popc(b);
    }
    int nnew = 0;
    for (int base = 0; base < sout; base += 32) {
      const int idx = base + lane;
      bool fresh = false;
      int child = 0;
      if (idx < sout) {
        int r = 0;
        while (r + 1 < nc && m.pout[r + 1] <= idx) ++r;
        const int y = m.outb[m.cs[r]] + idx - m.pout[r];
        child = __ldg(G.out_dst + y);
        // 16-bit counters decremented through their 32-bit word (a counter
        // is >= 1 when decremented, so no borrow crosses halves)
        unsigned *word = reinterpret_cast<unsigned *>(m.pending) + (child >> 1);
        const int sh = 16 * (child & 1);
        fresh = ((atomicSub(word, 1u << sh) >> sh) & 0xffffu) == 1;
      }
      const unsigned b = __ballot_sync(kFull, fresh);
      if (fresh) {
        const int at = nnew + __popc(b & ((1u << lane) - 1u));
        if (at < kSPairs) m.newn[at] = child;
      }
      nnew += __popc(b);
    }
    SMARK(P_COMMIT);
    // remove the committed slots, largest first (a moved-in last slot is never
    // a committed one)
    if (nc > 1) {
      if (lane < nc) {
        const int sr = m.cs[lane];
        int rank = 0;
        for (int r2 = 0; r2 < nc; ++r2) rank += m.cs[r2] > sr;
        m.ord[rank] = sr;
      }
    } else if (lane == 0) {
      m.ord[0] = m.cs[0];
    }
    __syncwarp();
    for (int r = 0; r < nc; ++r) {
      const int sc = m.ord[r], last = st.R - 1;
      if (sc != last) {
        // lanes move one field each
        if (lane < 10) {
          if (lane == 0) {
            const int nd = m.node[last];
            m.node[sc] = nd;
            m.rpos[nd] = sc;
          } else if (lane == 1) {
            m.need[sc] = m.need[last];
          } else {
            int32_t *f = lane == 2 ? m.kk : lane == 3 ? m.inb : lane == 4 ? m.ine : lane == 5 ? m.outb
                       : lane == 6 ? m.oute : lane == 7 ? m.alive : m.urg;
            if (lane < 9) f[sc] = f[last];
          }
        }
        if (lane < n) m.dr[sc * n + lane] = m.dr[last * n + lane];
      }
      --st.R;
      __syncwarp();
    }
    SMARK(P_REMOVE);
    // new ready slots
    const int R0 = st.R;
    st.R += nnew;
    if (st.R * n > kSPairs) {
      overflow = true;
      break;
    }
    for (int x = lane; x < nnew; x += 32) m.node[R0 + x] = m.newn[x];
    __syncwarp();
    small_fill_slots(m, G, R0, nnew, n - st.nexcl, lane);
    __syncwarp();
    // D: data-ready rows of the new slots ...
    for (int idx = lane; idx < nnew * n; idx += 32) {
      const int sl = idx / n, q = idx - sl * n, s = R0 + sl;
      int32_t urg = 0;
      if (m.excl[q]) {
        m.dr[s * n + q] = kSDead;
        if (kSct) small_dr<true>(m, G, n, m.inb[s], m.ine[s], q, urg);
      } else {
        m.dr[s * n + q] = small_dr<kSct>(m, G, n, m.inb[s], m.ine[s], q, urg);
      }
      if (kSct && q == 0) m.urg[s] = urg;
    }
    SMARK(P_ROWS);
    // ... and the consumers of each newly cached (producer, device) there
    for (int e0 = 0; e0 < nnc; e0 += 32) {
      const int ne = min(32, nnc - e0);
      int ob = 0, cnt = 0;
      if (lane < ne) {
        const int i = m.nci[e0 + lane];
        ob = __ldg(G.out_off + i);
        cnt = __ldg(G.out_off + i + 1) - ob;
      }
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(kFull, incl, o);
        if (lane >= o) incl += v;
      }
      const int tot = __shfl_sync(kFull, incl, 31);
      __syncwarp();
      m.pin[lane] = incl - cnt;  // free after phase A
      m.pout[lane] = ob;
      __syncwarp();
      for (int b0 = 0; b0 < tot; b0 += 32) {
        const int idx = b0 + lane;
        if (idx < tot) {
          int r = 0;
          while (r + 1 < ne && m.pin[r + 1] <= idx) ++r;
          const int p = m.ncp[e0 + r];
          const int c = __ldg(G.out_dst + m.pout[r] + idx - m.pin[r]);
          if (m.pending[c] == 0 && sm_dev(m.info[c]) < 0) {
            const int s = m.rpos[c];
            if (s >= 0 && m.dr[s * n + p] != kSDead) {
              int32_t urg;
              m.dr[s * n + p] = small_dr<false>(m, G, n, m.inb[s], m.ine[s], p, urg);
            }
          }
        }
      }
      __syncwarp();
    }
    __syncwarp();
    SMARK(P_CACHE);
  }
#undef SMARK

  if (overflow) return;  // the general kernel places it
  if (st.err_status) {
    if (lane == 0) {
      set_err(jb.err, st.err_status, st.err_code, st.err_node, 0);
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
  emit_exec_order(c, jb, m.scal, lane);
  if (lane == 0) {
    jb.stats[0] = st.discarded;
    jb.stats[1] = st.excluded;
    jb.stats[2] = st.awake;
    set_err(jb.err, kOk, E_NONE, 0, 0);
    *jb.sdone = 1;
    if (kProf && jb.prof) {
      prof[P_TOTAL] = clock64() - prof_t0;
      for (int k = 0; k < kProfSlots; ++k) jb.prof[k] = prof[k];
    }
  }
}

// ---- prep: int32 comm times and the non-uniform producers of a (graph, comm)
__global__ void k_prep_small(DGraph g, DPrep pr) {
  int bad = 0;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.E; x += gridDim.x * blockDim.x) {
    const int64_t c = pr.in_c[x];
    if (c < 0 || c >= (int64_t(1) << 30)) bad = 1;
    pr.in_c32[x] = static_cast<int32_t>(c);
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.V; i += gridDim.x * blockDim.x) {
    const int b = g.out_off[i], e = g.out_off[i + 1];
    bool uni = true;
    if (e > b) {
      const int64_t c0 = pr.in_c[g.inpos[b]];
      for (int y = b + 1; y < e && uni; ++y) uni = pr.in_c[g.inpos[y]] == c0;
    }
    pr.nu[i] = uni ? -1 : atomicAdd(pr.nu_count, 1);
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(pr.cbad, 1);
}

void launch_prep_small(const DGraph &g, const DPrep &pr, cudaStream_t s) {
  const int nb = ((g.V > g.E ? g.V : g.E) + 255) / 256;
  if (nb > 0) k_prep_small<<<nb < 1184 ? nb : 1184, 256, 0, s>>>(g, pr);
}

size_t small_smem_bytes_host(int V, int n, int nucap, int nccap) { return small_smem_bytes(V, n, nucap, nccap); }

// One CTA (one warp) per job; `order` lists the K2s jobs, m-ETF first.
template <bool kSct, bool kProf>
static void launch_sf(const DJob *jobs, const int32_t *order, int nj, const DGraph *graphs, const DPrep *preps,
                      size_t smem, cudaStream_t s) {
  if (nj <= 0) return;
  cudaFuncSetAttribute(k_place_small<kSct, kProf>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(smem));
  // the smallest shared-memory carveout that holds the job state: the rest
  // of the unified 256 KB is L1 for the warmed graph arrays
  const int pct = static_cast<int>((smem * 100 + 228 * 1024 - 1) / (228 * 1024));
  cudaFuncSetAttribute(k_place_small<kSct, kProf>, cudaFuncAttributePreferredSharedMemoryCarveout, pct < 1 ? 1 : pct);
  k_place_small<kSct, kProf><<<nj, 32 * kSWarm, smem, s>>>(jobs, order, nj, graphs, preps);
}

void launch_small_frontier(const DJob *jobs, const int32_t *order, int n_etf, int n_sct, const DGraph *graphs,
                           const DPrep *preps, size_t smem, bool prof, cudaStream_t s) {
  if (prof) {
    launch_sf<false, true>(jobs, order, n_etf, graphs, preps, smem, s);
    launch_sf<true, true>(jobs, order + n_etf, n_sct, graphs, preps, smem, s);
  } else {
    launch_sf<false, false>(jobs, order, n_etf, graphs, preps, smem, s);
    launch_sf<true, false>(jobs, order + n_etf, n_sct, graphs, preps, smem, s);
  }
}

}  // namespace bx

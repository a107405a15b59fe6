// K2s — the small-frontier list placer (parallel comm mode, m-ETF / m-SCT).
//
// Same contract as K2 (place_list, proj/src/placers.cpp:115-295, in its
// exact-argmin form): every step takes the lexicographic minimum of
// (key(j,p), j, p) over the live pairs and commits or discards it.
//
// Model-shaped training graphs keep a tiny ready frontier under list
// scheduling (Inception/GNMT/Transformer meta graphs: 3-12 ready nodes on
// average), so a placement is a chain of V dependent steps over a few dozen
// pairs, and its speed is the latency of one scheduling round. This kernel
// is built for that chain: ONE warp per problem, no CTA barriers, every
// mutable per-node value in shared memory, every live pair in a register of
// some lane (R * n <= 512, at most 16 pairs per lane), and the static graph
// read through packed records (one load per node, one per in-edge). Up to
// 32 devices (64 for m-ETF on graphs that need no cache rows).
//
// A round:
//   1. keys: each lane forms key = max(dev_free[q], DR[s][q]) (+ the m-SCT
//      awake floor, placers.cpp:147-156) for its pairs, as one 64-bit word
//      (key << 32 | node << 6 | q): (key, node, device) order in a single
//      unsigned compare; the memory check (placers.cpp:203-205) is a bit;
//   2. selection: a two-REDUX warp minimum gives the global argmin; a pair
//      that does not fit is discarded on the spot (placers.cpp:203-219);
//      a pair that fits commits. After committing (j, p) at t every key that
//      can change or appear is >= t + k_j (column p's keys are >= the new
//      dev_free[p]; a newly cached parent only touches column p; a newly
//      ready child has j as a parent), so the next minimum among the
//      untouched pairs commits in the same round while its key is below the
//      least such finish time T — at most one commit per device per round.
//      m-SCT: a lifted reservation may lower the keys of its column, which
//      then drops out of the round and lowers T to its dev_free (every key of
//      a column is >= its dev_free). A commit only updates registers here;
//   3. lane r applies commit r (dev_free, memory slack, finish, outputs);
//   4. one pass over the committed nodes' in- and out-edges: cache arrivals
//      of remote parents (commit_schedulable_time, placers.cpp:95-101) and
//      readiness (:256-268);
//   5. committed slots leave, the last live slots move into the holes (one
//      parallel step);
//   6. new slots: static fields and data-ready rows DR[s][q], one (slot,
//      device) item per lane;
//   7. re-keys of ready consumers whose parent tensor just landed on a
//      device (:271-279).
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
// for the m-SCT floor), 0 <= c < 2^16 - 1, in-degrees below 2^16 - 1 and
// V < 2^16 - 1 (16-bit counters and packed indices). Any check that fails —
// or a frontier beyond 512 pairs at any point — leaves sdone = 0 and the
// general kernels (listsched.cu), launched behind this one, place the job
// instead.
//
// Per-node state is 12 bytes of shared memory (finish/device, pending,
// ready slot), so graphs up to ~12k meta nodes fit; the rest of the SM's
// 256 KB is L1, which three helper warps fill with the packed graph before
// the scheduling warp needs it.
#include "sched_common.cuh"

namespace bx {

constexpr int kSP = 16;                  // pairs per lane
constexpr int kSPairs = 32 * kSP;        // R * n <= 512
constexpr int kSDev = 64;                // devices (m-ETF on graphs without cache rows; m-SCT and
                                         // graphs with non-uniform producers: 32)
constexpr int kSDevBits = 6;             // device field of a packed pair
constexpr int kSSlots = kSPairs;         // newly-ready list capacity
constexpr int kKI = 8;                   // parents cached per ready slot (in_pack records)
constexpr int kKO = 8;                   // children cached per ready slot
// ready-slot capacity for n devices (R * n <= kSPairs)
__host__ __device__ inline int small_slots(int n) { return kSPairs / (n > 0 ? n : 1); }
constexpr int32_t kSDead = 0x7fffffff;   // DR of a discarded / excluded pair
constexpr uint64_t kSNone = ~0ull;

__device__ __forceinline__ uint64_t sm_min_u64(uint64_t v) {
  const unsigned hi = static_cast<unsigned>(v >> 32), lo = static_cast<unsigned>(v);
  const unsigned mhi = __reduce_min_sync(kFull, hi);
  const unsigned mlo = __reduce_min_sync(kFull, hi == mhi ? lo : 0xffffffffu);
  return (static_cast<uint64_t>(mhi) << 32) | mlo;
}

__device__ __forceinline__ int sm_dev(uint64_t info) { return static_cast<int>(static_cast<uint32_t>(info)); }
__device__ __forceinline__ int32_t sm_fin(uint64_t info) { return static_cast<int32_t>(info >> 32); }

// New-arrival bitset over (non-uniform producer, device): words, one spare
// so a producer's n bits can always be read as a 64-bit window.
__host__ __device__ inline int small_ncm_words(int nucap, int n) { return (nucap * n + 31) / 32 + 1; }
__device__ __forceinline__ uint32_t ncm_bits(const uint32_t *w, int u, int n) {
  const int b = u * n;
  const uint64_t v = (static_cast<uint64_t>(w[(b >> 5) + 1]) << 32 | w[b >> 5]) >> (b & 31);
  return static_cast<uint32_t>(v) & (n >= 32 ? ~0u : (1u << n) - 1u);
}
__device__ __forceinline__ void ncm_clear(uint32_t *w, int u, int n) {
  const int b = u * n;
  const uint64_t m = (n >= 32 ? 0xffffffffull : (1ull << n) - 1ull) << (b & 31);
  atomicAnd(w + (b >> 5), ~static_cast<uint32_t>(m));
  if (m >> 32) atomicAnd(w + (b >> 5) + 1, ~static_cast<uint32_t>(m >> 32));
}

// Shared-memory layout of one problem (host: small_smem_bytes).
struct SSm {
  int32_t *F, *awf, *awu, *excl;  // [kSDev] per device
  int64_t *slack;                 // [kSDev] capacity - reserved
  uint64_t *info;                 // [V] finish << 32 | device (0xffffffff: unplaced)
  uint16_t *pending;              // [V] parents not yet placed (decremented as 32-bit words)
  int16_t *rpos;                  // [V] ready slot of a node, -1 none
  uint16_t *nuc;                  // [nucap * n] per non-uniform producer and device: comm time of the
                                  // edge that first brought its tensor there (arrival = finish + it), 0xffff absent
  // ready slots (ns = small_slots(n))
  int32_t *node, *kk, *inb, *outb, *cnt, *alive, *urg, *favs;  // [ns]; cnt = in_cnt | out_cnt << 16; favs: m-SCT favourite
  int64_t *need;                                        // [ns]
  uint2 *sip;                                           // [ns * kKI] the slot's first parents (in_pack records)
  int32_t *sco;                                         // [ns * kKO] the slot's first children
  int32_t *dr;                                          // [kSPairs] DR[s * n + q]
  int32_t *cjs;                                         // [32] the round's commits so far (lane 0)
  // per round
  int32_t *pin, *pout;  // [32] per commit: first in- / out-edge item
  int32_t *cpd, *csl;   // [32] per commit: device, slot
  int32_t *ita, *itb;   // [32] per in-item of a 32-item chunk: slot << 16 | k, device
  int32_t *ito;         // [32] per out-item: slot << 16 | k
  int32_t *nci;         // [nccap] non-uniform producers newly cached this round (nu index)
  uint32_t *ncm;        // bit u * n + p: non-uniform producer u newly reached device p this round
  int32_t *newn;        // [kSSlots] newly ready nodes
  int32_t *scal;        // [kSDev] exec-order counters
};

__host__ __device__ inline size_t small_smem_bytes(int V, int n, int nucap, int nccap) {
  size_t b = 0;
  b += kSDev * 8 + 4 * kSDev * 4;                              // slack, F/awf/awu/excl
  b += size_t(V) * 8 + 2 * ((size_t(V) * 2 + 3) & ~size_t(3)); // info, pending, rpos
  b += (size_t(nucap) * n * 2 + 7) & ~size_t(7);               // nuc
  const size_t ns = static_cast<size_t>(small_slots(n));
  b += ns * (8 * 4 + 8 + 8 * kKI + 4 * kKO) + size_t(kSPairs) * 4 + 32 * 4;  // slots, caches, dr, cjs
  b += 7 * 32 * 4 + size_t(nccap) * 4 + small_ncm_words(nucap, n) * 4 + size_t(kSSlots) * 4 + kSDev * 4;
  return b + 64;
}

// Node state in HBM: the pending counts still fit shared memory as bytes
// (one word holds four) when every in-degree is below 256 and the slot tables
// plus V bytes stay within kSPendMax; the extra bytes past the slot tables, or 0.
constexpr size_t kSPendMax = 200 * 1024;
__host__ __device__ inline size_t small_pend_bytes(int V, int n, int nucap, int nccap, int maxin) {
  const size_t base = (small_smem_bytes(0, n, nucap, nccap) + 15) & ~size_t(15);
  const size_t extra = base - small_smem_bytes(0, n, nucap, nccap) + ((static_cast<size_t>(V) + 3) & ~size_t(3));
  return maxin < 256 && small_smem_bytes(0, n, nucap, nccap) + extra <= kSPendMax ? extra : 0;
}

__device__ __forceinline__ SSm small_layout(unsigned char *base, int V, int n, int nucap, int nccap) {
  SSm m;
  int64_t *p64 = reinterpret_cast<int64_t *>(base);
  m.slack = p64;
  m.info = reinterpret_cast<uint64_t *>(p64 + kSDev);
  const int ns = small_slots(n);
  m.need = reinterpret_cast<int64_t *>(m.info + V);
  m.sip = reinterpret_cast<uint2 *>(m.need + ns);
  int32_t *p32 = reinterpret_cast<int32_t *>(m.sip + ns * kKI);
  m.F = p32;
  m.awf = p32 + kSDev;
  m.awu = p32 + 2 * kSDev;
  m.excl = p32 + 3 * kSDev;
  p32 += 4 * kSDev;
  const int vw = (V + 1) / 2;  // int32 words of a [V] 16-bit array
  m.pending = reinterpret_cast<uint16_t *>(p32);
  m.rpos = reinterpret_cast<int16_t *>(p32 + vw);
  p32 += 2 * vw;
  m.nuc = reinterpret_cast<uint16_t *>(p32);
  p32 += (nucap * n + 1) / 2;
  m.node = p32;
  m.kk = p32 + ns;
  m.inb = p32 + 2 * ns;
  m.outb = p32 + 3 * ns;
  m.cnt = p32 + 4 * ns;
  m.alive = p32 + 5 * ns;
  m.urg = p32 + 6 * ns;
  m.favs = p32 + 7 * ns;
  p32 += 8 * ns;
  m.sco = p32;
  p32 += ns * kKO;
  m.dr = p32;
  p32 += kSPairs;
  m.cjs = p32;
  p32 += 32;
  m.pin = p32;
  m.pout = p32 + 32;
  m.cpd = p32 + 64;
  m.csl = p32 + 96;
  m.ita = p32 + 128;
  m.itb = p32 + 160;
  m.ito = p32 + 192;
  p32 += 224;
  m.nci = p32;
  m.ncm = reinterpret_cast<uint32_t *>(p32 + nccap);
  m.newn = p32 + nccap + small_ncm_words(nucap, n);
  m.scal = m.newn + kSSlots;
  return m;
}

// Read-only packed graph (global memory, read through the non-coherent path).
struct SGraph {
  const int4 *__restrict__ node;    // [2V] in_b, out_b, in_cnt | out_cnt << 16, k; need (int64), 0, 0
  const uint2 *__restrict__ inp;    // [E] per in-CSR slot: parent, (nu(parent) + 1) << 16 | c
  const int32_t *__restrict__ out_dst;
  const int32_t *__restrict__ fav;
  const int64_t *__restrict__ need;
  const int32_t *__restrict__ need_order;
};

// Parent k of ready slot s (its in_pack record): the slot cache for the
// first kKI, the packed graph beyond.
__device__ __forceinline__ uint2 slot_parent(const SSm &m, const SGraph &G, int s, int k) {
  return k < kKI ? m.sip[s * kKI + k] : __ldg(G.inp + m.inb[s] + k);
}

__device__ __forceinline__ int slot_child(const SSm &m, const SGraph &G, int s, int k) {
  return k < kKO ? m.sco[s * kKO + k] : __ldg(G.out_dst + m.outb[s] + k);
}

// One parent's term of DR on device q (placers.cpp:55-61), and its
// urgency term.
__device__ __forceinline__ int32_t parent_term(const SSm &m, int n, uint2 a, int q, int32_t &urg_term) {
  const uint64_t ia = m.info[a.x];
  const int32_t ca = static_cast<int32_t>(a.y & 0xffffu);
  const int ua = static_cast<int>(a.y >> 16) - 1;
  const int32_t fa = sm_fin(ia);
  const unsigned za = ua >= 0 ? m.nuc[ua * n + q] : 0xffffu;
  urg_term = fa + ca;
  return sm_dev(ia) == q ? fa : fa + (za != 0xffffu ? static_cast<int32_t>(za) : ca);
}

// DR of ready slot s on device q from its cached parents (and urgency).
template <bool kUrg>
__device__ __forceinline__ int32_t slot_dr(const SSm &m, const SGraph &G, int n, int s, int indeg, int q,
                                           int32_t &urg) {
  int32_t t = 0, u = 0;
  for (int k = 0; k < indeg; ++k) {
    int32_t ut;
    t = max(t, parent_term(m, n, slot_parent(m, G, s, k), q, ut));
    if (kUrg) u = max(u, ut);
  }
  urg = u;
  return t;
}

// Per-problem loop state kept in registers (identical in every lane).
struct SRun {
  int R, placed, nexcl, minptr;
  int64_t discarded, excluded, awake;
  int err_status, err_code, err_node;
  int32_t cmax;
  int V, n, d32, r32, s0, q0;
};

// One round's commits, lane r holding commit r.
struct SCommit {
  int nc;
  int j, p, s;
  int32_t t, fin;
};

// Node j committed earlier in this round (not yet applied to `info`; the
// selection lists the round's commits in m.cjs).
__device__ __forceinline__ bool committed_now(const SSm &m, int nc, int j) {
  bool done = false;
  for (int r = 0; r < nc; ++r) done |= m.cjs[r] == j;
  return done;
}

// Steps 1-2 of a round with P pairs per lane (R * n <= 32 P): keys, then
// exact commits / discards below the threshold. Returns false when no live
// pair exists at all.
template <int P, bool kSct>
__device__ __forceinline__ bool small_select(const SSm &m, const SGraph &G, SRun &st, int lane, SCommit &cm) {
  const int n = st.n;
  const int np = st.R * n;
  uint64_t ck[P];
  int32_t kq[P];  // k of the pair's node
  int32_t sq[P];  // slot << kSDevBits | device
  unsigned fitm = 0;
  {
    int s = st.s0, q = st.q0;
#pragma unroll
    for (int u = 0; u < P; ++u) {
      const int x = lane + 32 * u;
      ck[u] = kSNone;
      kq[u] = 0;
      sq[u] = s << kSDevBits | q;
      if (x < np) {
        const int32_t d = m.dr[x];
        if (d != kSDead && !m.excl[q]) {
          const int node = m.node[s];
          int32_t key = max(m.F[q], d);
          if (kSct) {  // the three loads issue together
            const int a = m.awf[q];
            const int32_t fl = min(m.awu[q], m.urg[s]);
            if (a >= 0 && a != node) key = max(key, fl);
          }
          ck[u] = (static_cast<uint64_t>(static_cast<uint32_t>(key)) << 32) |
                  (static_cast<uint32_t>(node) << kSDevBits | static_cast<uint32_t>(q));
          kq[u] = m.kk[s];
          if (m.need[s] <= m.slack[q]) fitm |= 1u << u;
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
  __syncwarp();  // every lane's key reads precede the selection's shared-memory writes
  uint32_t T = 0xffffffffu;
  cm.nc = 0;
  bool progress = false;
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
    const int j = static_cast<int>((static_cast<uint32_t>(w)) >> kSDevBits);
    const int p = static_cast<int>(w & (kSDev - 1u));
    const int s = (msq >> kSDevBits) & 0xffffff;
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
        return true;
      }
      ++st.discarded;
      // smallest need among all unplaced nodes (the `remaining` multiset);
      // column p has no commit this round, so its slack is current
      int64_t minrem = 0;
      if (lane == 0) {
        int x;
        while (x = __ldg(G.need_order + st.minptr), sm_dev(m.info[x]) >= 0 || committed_now(m, cm.nc, x))
          ++st.minptr;
        minrem = __ldg(G.need + x);
      }
      minrem = __shfl_sync(kFull, minrem, 0);
      if (minrem > m.slack[p]) {
        // exclusion: every unplaced (j2, p) dies (ascending j2 in the
        // reference; the first node left with no device is the smallest)
        ++st.excluded;
        ++st.nexcl;
        int first_dead = INT32_MAX;
        for (int s2 = lane; s2 < st.R; s2 += 32) {
          const int node2 = m.node[s2];
          if (sm_dev(m.info[node2]) >= 0 || committed_now(m, cm.nc, node2)) continue;
          const int x2 = s2 * n + p;
          if (m.dr[x2] != kSDead) {
            m.dr[x2] = kSDead;
            if (--m.alive[s2] == 0) first_dead = min(first_dead, node2);
          }
        }
        if (st.nexcl == n)  // no device left: the smallest unplaced node is the casualty
          for (int x = lane; x < st.V; x += 32)
            if (sm_dev(m.info[x]) < 0 && !committed_now(m, cm.nc, x)) first_dead = min(first_dead, x);
        first_dead = static_cast<int>(__reduce_min_sync(kFull, static_cast<unsigned>(first_dead)));
        if (first_dead != INT32_MAX) {
          st.err_status = kInfeasible;
          st.err_code = E_FITS_NONE;
          st.err_node = first_dead;
          return true;
        }
        if (lane == 0) m.excl[p] = 1;
#pragma unroll
        for (int u = 0; u < P; ++u)
          if ((sq[u] & (kSDev - 1)) == p) ck[u] = kSNone;
      }
      __syncwarp();
      continue;
    }
    // ---- commit (placers.cpp:221-233): registers only; step 3 applies it ----
    const int32_t fin = t + mk;
    if (lane == cm.nc) {
      cm.j = j;
      cm.p = p;
      cm.s = s;
      cm.t = t;
      cm.fin = fin;
    }
    if (lane == 0) m.cjs[cm.nc] = j;
    ++cm.nc;
    ++st.placed;
    T = min(T, static_cast<uint32_t>(fin));
#pragma unroll
    for (int u = 0; u < P; ++u)
      if ((sq[u] & (kSDev - 1)) == p || (static_cast<uint32_t>(ck[u]) >> kSDevBits) == static_cast<uint32_t>(j))
        ck[u] = kSNone;
    if (kSct) {
      // awake reservations (placers.cpp:235-254): columns whose reservation
      // awaited j are lifted — their keys may drop, so they leave the round
      // and bound it by their dev_free (the one before this round's commit
      // on that column, if any: smaller, so only more conservative)
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
        if ((lm >> (sq[u] & (kSDev - 1))) & 1) ck[u] = kSNone;  // m-SCT: n <= 32
      int got = 0;
      if (lane == 0) {
        m.awf[p] = -1;
        const int h = m.favs[s];  // the committed slot's favourite (loaded with the slot)
        // h unplaced: not placed before this round and not committed in it
        if (h >= 0 && sm_dev(m.info[h]) < 0 && !committed_now(m, cm.nc, h)) {
          m.awf[p] = h;
          m.awu[p] = fin + st.cmax;
          got = 1;
        }
      }
      st.awake += __shfl_sync(kFull, got, 0);
      __syncwarp();
    }
    if (st.placed == st.V || cm.nc == 32) break;  // lane r holds commit r (n may reach 64)
  }
  __syncwarp();  // ... and the commits' writes (step 3) follow every lane's reads
  return progress;
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
// packed graph the scheduler reads into the SM's L1, then exit.
constexpr int kSWarm = 4;

// kGlobal: graphs whose per-node state does not fit one SM's shared memory
// (the reference's layered-chain at 100k nodes, 16 chains, ...): finish /
// device, pending counts and ready slots live in the job's HBM scratch
// (L1/L2-resident), the ready slots, column caches and key rows stay in
// shared memory, and the graph is not pre-warmed.
template <bool kSct, bool kProf, bool kGlobal>
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
    if (kGlobal) return;
    const int tid = threadIdx.x - 32, nt = 32 * (kSWarm - 1);
    const size_t V = static_cast<size_t>(g.V), E = static_cast<size_t>(g.E);
    unsigned acc = warm_l1(pr.node_pack, 16 * V, tid, nt) ^ warm_l1(pr.in_pack, 8 * E, tid, nt);
    acc ^= warm_l1(g.need, 8 * V, tid, nt);
    acc ^= warm_l1(g.edst, 4 * E, tid, nt);
    // (need_order is read only when a pair is discarded: not warmed)
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
  const int nccap = n * (jb.maxin > 1 ? jb.maxin : 1);
  // dynamic eligibility (see the header); otherwise the general kernel runs it
  if (*pr.cbad || g.flags[2] || *g.ksum < 0 || *pr.nu_count > jb.nucap || n > kSDev ||
      (n > 32 && (kSct || *pr.nu_count > 0)) || V >= (kGlobal ? (1 << 26) : 0xffff) ||
      cmax64 >= 0xffff || jb.maxin >= 0xffff || *g.ksum + (int64_t(V) + 2) * cmax64 >= int64_t(INT32_MAX))
    return;
  const int32_t cmax = static_cast<int32_t>(cmax64);
  SSm m = small_layout(smem, kGlobal ? 0 : V, n, jb.nucap, nccap);
  // kGlobal: pending counts as bytes in shared memory when they fit
  uint32_t *pend8 = nullptr;
  if (kGlobal && small_pend_bytes(V, n, jb.nucap, nccap, jb.maxin) > 0)
    pend8 = reinterpret_cast<uint32_t *>(smem + ((small_smem_bytes(0, n, jb.nucap, nccap) + 15) & ~size_t(15)));
  if (kGlobal) {
    m.info = reinterpret_cast<uint64_t *>(jb.finish);    // [V] int64
    m.pending = reinterpret_cast<uint16_t *>(jb.pending);  // [V] int32 words hold 2V halves
    m.rpos = reinterpret_cast<int16_t *>(jb.rpos);
  }
  SGraph G;
  G.node = pr.node_pack;
  G.inp = pr.in_pack;
  G.out_dst = g.edst;
  G.fav = jb.fav;
  G.need = g.need;
  G.need_order = g.need_order;

  // ---- init ------------------------------------------------------------------
  {
    for (int d = lane; d < kSDev; d += 32) {
      m.F[d] = 0;
      m.awf[d] = -1;
      m.awu[d] = 0;
      m.excl[d] = 0;
      m.slack[d] = d < n ? jb.cap[d] : 0;
    }
    for (int x = lane; x < jb.nucap * n; x += 32) m.nuc[x] = 0xffffu;
    for (int x = lane; x < small_ncm_words(jb.nucap, n); x += 32) m.ncm[x] = 0;
  }
  int R = 0;
  for (int base = 0; base < V; base += 32) {
    const int j = base + lane;
    bool src = false;
    if (j < V) {
      const int4 nd = __ldg(G.node + j);
      const int indeg = nd.z & 0xffff;
      m.info[j] = 0xffffffffull;
      if (kGlobal && pend8)
        reinterpret_cast<uint8_t *>(pend8)[j] = static_cast<uint8_t>(indeg);
      else
        m.pending[j] = static_cast<uint16_t>(indeg);
      m.rpos[j] = -1;
      src = indeg == 0;
    }
    const unsigned b = __ballot_sync(kFull, src);
    if (src) {
      const int s = R + __popc(b & ((1u << lane) - 1u));
      if (s < kSSlots) m.newn[s] = j;
    }
    R += __popc(b);
  }
  if (R * n > kSPairs) return;  // frontier too wide from the start
  __syncwarp();

  SRun st;
  st.R = 0;
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

  int nnew = R;  // the sources are the first "newly ready" nodes
  bool overflow = false;
  SCommit cm;
  cm.nc = 0;
  cm.j = cm.p = cm.s = 0;
  cm.t = cm.fin = 0;
  while (true) {
    // ---- 6. new slots: statics, parent / child caches, data-ready rows ---------
    {
      const int R0 = st.R;
      st.R += nnew;
      if (st.R * n > kSPairs) {
        overflow = true;
        break;
      }
      const int alive0 = n - st.nexcl;
      // 6a. one lane per new slot: the packed node record, then its first
      // kKI parents and kKO children (independent loads, issued together);
      // the children's records are prefetched for when they become ready
      for (int sl = lane; sl < nnew; sl += 32) {
        const int s = R0 + sl;
        const int c = m.newn[sl];
        const int4 nd = __ldg(G.node + c);
        const int64_t nneed = __ldg(G.need + c);
        const int ci = nd.z & 0xffff, co = nd.z >> 16;
        uint2 pa[kKI];
        int ch[kKO];
#pragma unroll
        for (int k = 0; k < kKI; ++k)
          if (k < ci) pa[k] = __ldg(G.inp + nd.x + k);
#pragma unroll
        for (int k = 0; k < kKO; ++k)
          if (k < co) ch[k] = __ldg(G.out_dst + nd.y + k);
        m.node[s] = c;
        m.rpos[c] = static_cast<int16_t>(s);
        m.kk[s] = nd.w;
        m.inb[s] = nd.x;
        m.outb[s] = nd.y;
        m.cnt[s] = nd.z;
        m.alive[s] = alive0;
        if (kSct) m.favs[s] = __ldg(G.fav + c);
        m.need[s] = nneed;
#pragma unroll
        for (int k = 0; k < kKI; ++k)
          if (k < ci) m.sip[s * kKI + k] = pa[k];
#pragma unroll
        for (int k = 0; k < kKO; ++k)
          if (k < co) {
            m.sco[s * kKO + k] = ch[k];
            asm volatile("prefetch.global.L1 [%0];" ::"l"(G.node + ch[k]));
          }
      }
      __syncwarp();
      // 6b. data-ready rows: item idx = lane + 32 k -> (slot sl, device q)
      int sl = st.s0, q = st.q0;
      for (int idx = lane; idx < nnew * n; idx += 32) {
        const int s = R0 + sl;
        const int ci = m.cnt[s] & 0xffff;
        int32_t urg = 0;
        int32_t d;
        if (m.excl[q]) {
          d = kSDead;
          if (kSct) slot_dr<true>(m, G, n, s, ci, q, urg);
        } else {
          d = slot_dr<kSct>(m, G, n, s, ci, q, urg);
        }
        m.dr[s * n + q] = d;
        if (q == 0) m.urg[s] = urg;
        sl += st.d32;
        q += st.r32;
        if (q >= n) {
          q -= n;
          ++sl;
        }
      }
      __syncwarp();
    }
    SMARK(P_ROWS);
    if (st.placed == V) break;

    // ---- 1-2. keys and the round's exact commits ------------------------------
    const int np = st.R * n;
    const bool progress = np <= 32    ? small_select<1, kSct>(m, G, st, lane, cm)
                          : np <= 64  ? small_select<2, kSct>(m, G, st, lane, cm)
                          : np <= 128 ? small_select<4, kSct>(m, G, st, lane, cm)
                          : np <= 256 ? small_select<8, kSct>(m, G, st, lane, cm)
                                      : small_select<16, kSct>(m, G, st, lane, cm);
    const int nc = cm.nc;
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
    nnew = 0;
    if (nc == 0) continue;

    // ---- 3. apply the commits (one device each) -------------------------------
    int cin = 0, cout = 0;
    if (lane < nc) {
      const int p = cm.p, s = cm.s, j = cm.j;
      m.F[p] = cm.fin;
      m.slack[p] -= m.need[s];
      m.info[j] = (static_cast<uint64_t>(static_cast<uint32_t>(cm.fin)) << 32) | static_cast<uint32_t>(p);
      jb.device_of[j] = p;
      jb.start[j] = cm.t;
      jb.cseq[st.placed - nc + lane] = j;
      const int c2 = m.cnt[s];
      cin = c2 & 0xffff;
      cout = c2 >> 16;
    }
    // per-commit first item (inclusive scan of the packed counts)
    int incl = cin | (cout << 16);
    for (int o = 1; o < nc; o <<= 1) {  // lanes >= nc hold 0 and are never read below
      const int v = __shfl_up_sync(kFull, incl, o);
      if (lane >= o) incl += v;
    }
    const int tot = __shfl_sync(kFull, incl, nc - 1);
    const int tin = tot & 0xffff, tout = tot >> 16;
    const int pin = (incl & 0xffff) - cin, pout = (incl >> 16) - cout;
    SMARK(P_COMMIT);

    // ---- 4. cache arrivals (every in-edge of a committed node) and readiness
    // (every out-edge), one pass: 32-item chunks of both lists side by side;
    // each commit lane writes its items into the chunk tables, then lane i
    // takes in-item base + i and out-item base + i (two independent chains)
    int nnc = 0;
    const int titems = max(tin, tout);
    for (int base = 0; base < titems; base += 32) {
      if (lane < nc) {
        const int ilo = max(pin, base), ihi = min(pin + cin, base + 32);
        const int olo = max(pout, base), ohi = min(pout + cout, base + 32);
        for (int k = ilo; k < ihi; ++k) {
          m.ita[k - base] = cm.s << 16 | (k - pin);
          m.itb[k - base] = cm.p;
        }
        for (int k = olo; k < ohi; ++k) m.ito[k - base] = cm.s << 16 | (k - pout);
      }
      __syncwarp();
      bool fresh = false, ready = false;
      int a = 0, child = 0;
      const bool hin = base + lane < tin, hout = base + lane < tout;
      const int iti = m.ita[lane], itp = m.itb[lane], ito = m.ito[lane];
      if (hout) {
        child = slot_child(m, G, ito >> 16, ito & 0xffff);
        // 16-bit counters decremented through their 32-bit word (a counter
        // is >= 1 when decremented, so no borrow crosses halves)
        if (kGlobal && pend8) {  // bytes in shared memory, four to a word (same no-borrow argument)
          const int sh = 8 * (child & 3);
          ready = ((atomicSub(pend8 + (child >> 2), 1u << sh) >> sh) & 0xffu) == 1;
        } else {
          unsigned *word = reinterpret_cast<unsigned *>(m.pending) + (child >> 1);
          const int sh = 16 * (child & 1);
          ready = ((atomicSub(word, 1u << sh) >> sh) & 0xffffu) == 1;
        }
        if (ready) asm volatile("prefetch.global.L1 [%0];" ::"l"(G.node + child));
      }
      if (hin) {
        const uint2 e = slot_parent(m, G, iti >> 16, iti & 0xffff);
        const int u = static_cast<int>(e.y >> 16) - 1;
        if (u >= 0 && sm_dev(m.info[e.x]) != itp) {
          // one commit per device per round, so no two lanes share a slot
          uint16_t *slot = m.nuc + u * n + itp;
          if (*slot == 0xffffu) {
            *slot = static_cast<uint16_t>(e.y & 0xffffu);
            const int bit = u * n + itp;
            atomicOr(m.ncm + (bit >> 5), 1u << (bit & 31));
            fresh = true;  // u may be listed twice (two commits of the round share it)
            a = u;
          }
        }
      }
      const unsigned bf = __ballot_sync(kFull, fresh), br = __ballot_sync(kFull, ready);
      if (fresh) m.nci[nnc + __popc(bf & ((1u << lane) - 1u))] = a;
      if (ready) {
        const int at = nnew + __popc(br & ((1u << lane) - 1u));
        if (at < kSSlots) m.newn[at] = child;
      }
      nnc += __popc(bf);
      nnew += __popc(br);
      __syncwarp();
    }
    SMARK(P_READY);

    // ---- 5. remove the committed slots -----------------------------------------
    // holes = committed slots below the new end R'; movers = live slots in
    // [R', R); the i-th hole takes the i-th mover
    {
      const int Rn = st.R - nc;
      const bool committed_lane = lane < nc;
      const int cs = committed_lane ? cm.s : -1;
      const bool hole = committed_lane && cs < Rn;
      const unsigned tailmask = __reduce_or_sync(kFull, committed_lane && cs >= Rn ? 1u << (cs - Rn) : 0u);
      const unsigned live_tail = ~tailmask & ((nc >= 32) ? 0xffffffffu : ((1u << nc) - 1u));
      const unsigned hb = __ballot_sync(kFull, hole);
      const int nholes = __popc(hb);
      if (hole) {
        const int rank = __popc(hb & ((1u << lane) - 1u));
        const int src = Rn + static_cast<int>(__fns(live_tail, 0, rank + 1));
        m.pin[rank] = cs;  // hole / mover pairs for the cache copies below
        m.pout[rank] = src;
        const int nd = m.node[src];
        m.node[cs] = nd;
        m.rpos[nd] = static_cast<int16_t>(cs);
        m.need[cs] = m.need[src];
        m.kk[cs] = m.kk[src];
        m.inb[cs] = m.inb[src];
        m.outb[cs] = m.outb[src];
        m.cnt[cs] = m.cnt[src];
        m.alive[cs] = m.alive[src];
        m.urg[cs] = m.urg[src];
        if (kSct) m.favs[cs] = m.favs[src];
        for (int q = 0; q < n; ++q) m.dr[cs * n + q] = m.dr[src * n + q];
      }
      if (committed_lane) m.rpos[cm.j] = -1;
      st.R = Rn;
      __syncwarp();
      // the movers' parent / child caches, kKI + kKO words per pair of slots
      for (int it = lane; it < nholes * (kKI + kKO); it += 32) {
        const int h = it / (kKI + kKO), k = it - h * (kKI + kKO);
        const int dst = m.pin[h], src = m.pout[h];
        if (k < kKI) m.sip[dst * kKI + k] = m.sip[src * kKI + k];
        else m.sco[dst * kKO + k - kKI] = m.sco[src * kKO + k - kKI];
      }
      __syncwarp();
    }
    SMARK(P_REMOVE);
    if (nnew > kSSlots || (st.R + nnew) * n > kSPairs) {
      overflow = true;
      break;
    }

    // ---- 7. ready consumers of each newly cached (producer, device) re-key ----
    // one lane per ready slot ORs its non-uniform parents' new-arrival device
    // masks (step 4a) and re-keys those columns; the masks are then cleared
    if (nnc > 0) {
      for (int s = lane; s < st.R; s += 32) {
        const int ci = m.cnt[s] & 0xffff;
        uint32_t rk = 0;
        for (int k = 0; k < ci; ++k) {
          const int u = static_cast<int>(slot_parent(m, G, s, k).y >> 16) - 1;
          if (u >= 0) rk |= ncm_bits(m.ncm, u, n);
        }
        while (rk) {
          const int p = __ffs(rk) - 1;
          rk &= rk - 1;
          if (m.dr[s * n + p] != kSDead) {
            int32_t urg;
            m.dr[s * n + p] = slot_dr<false>(m, G, n, s, ci, p, urg);
          }
        }
      }
      __syncwarp();
      for (int e = lane; e < nnc; e += 32) ncm_clear(m.ncm, m.nci[e], n);
      __syncwarp();
    }
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

// ---- prep: the packed graph and the non-uniform producers of a (graph, comm)
__global__ void k_prep_small(DGraph g, DPrep pr) {
  int bad = 0;
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.E; x += gridDim.x * blockDim.x) {
    const int64_t c = pr.in_c[x];
    if (c < 0 || c >= 0xffff) bad = 1;
  }
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < g.V; i += gridDim.x * blockDim.x) {
    const int b = g.out_off[i], e = g.out_off[i + 1];
    bool uni = true;
    if (e > b) {
      const int64_t c0 = pr.in_c[g.inpos[b]];
      for (int y = b + 1; y < e && uni; ++y) uni = pr.in_c[g.inpos[y]] == c0;
    }
    pr.nu[i] = uni ? -1 : atomicAdd(pr.nu_count, 1);
    const int ib = g.in_off[i], ie = g.in_off[i + 1];
    const int64_t k = g.k[i];
    pr.node_pack[i] = make_int4(ib, b, (ie - ib) | ((e - b) << 16), static_cast<int32_t>(k));
  }
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) atomicOr(pr.cbad, 1);
}

// in_pack needs every producer's nu index (the kernel above), so it is a
// second pass
__global__ void k_prep_small_in(DGraph g, DPrep pr) {
  for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < g.E; x += gridDim.x * blockDim.x) {
    const int i = g.in_src[x];
    const int64_t c = pr.in_c[x];
    const unsigned nu1 = static_cast<unsigned>(pr.nu[i] + 1);
    pr.in_pack[x] = make_uint2(static_cast<unsigned>(i), (nu1 << 16) | static_cast<unsigned>(c & 0xffff));
  }
}

void launch_prep_small(const DGraph &g, const DPrep &pr, cudaStream_t s) {
  const int nb = ((g.V > g.E ? g.V : g.E) + 255) / 256;
  if (nb > 0) {
    k_prep_small<<<nb < 1184 ? nb : 1184, 256, 0, s>>>(g, pr);
    k_prep_small_in<<<nb < 1184 ? nb : 1184, 256, 0, s>>>(g, pr);
  }
}

size_t small_smem_bytes_host(int V, int n, int nucap, int nccap) { return small_smem_bytes(V, n, nucap, nccap); }
size_t small_pend_bytes_host(int V, int n, int nucap, int nccap, int maxin) {
  return small_pend_bytes(V, n, nucap, nccap, maxin);
}

// One CTA per job; `order` lists the K2s jobs, m-ETF first.
template <bool kSct, bool kProf, bool kGlobal>
static void launch_sf(const DJob *jobs, const int32_t *order, int nj, const DGraph *graphs, const DPrep *preps,
                      size_t smem, cudaStream_t s) {
  if (nj <= 0) return;
  auto kern = k_place_small<kSct, kProf, kGlobal>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
  // shared memory: the smallest carveout that holds the job state (the rest
  // of the unified 256 KB is L1 for the warmed graph); node state in HBM:
  // no warm-up warps, one warp per CTA, room for up to 8 CTAs per SM (the
  // register budget's limit)
  const size_t per_sm = kGlobal ? 8 * smem : smem;
  const int pct = static_cast<int>((per_sm * 100 + 228 * 1024 - 1) / (228 * 1024));
  cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout, pct < 1 ? 1 : (pct > 100 ? 100 : pct));
  kern<<<nj, kGlobal ? 32 : 32 * kSWarm, smem, s>>>(jobs, order, nj, graphs, preps);
}

// `order` lists the K2s jobs in four runs: m-ETF and m-SCT with shared-memory
// node state, then m-ETF and m-SCT with global node state (counts cnt[4],
// shared-memory bytes smem[2]: per-node-state and global variants).
void launch_small_frontier(const DJob *jobs, const int32_t *order, const int *cnt, const DGraph *graphs,
                           const DPrep *preps, const size_t *smem, bool prof, cudaStream_t s) {
  const int32_t *o1 = order + cnt[0], *o2 = o1 + cnt[1], *o3 = o2 + cnt[2];
  if (prof) {
    launch_sf<false, true, false>(jobs, order, cnt[0], graphs, preps, smem[0], s);
    launch_sf<true, true, false>(jobs, o1, cnt[1], graphs, preps, smem[0], s);
    launch_sf<false, true, true>(jobs, o2, cnt[2], graphs, preps, smem[1], s);
    launch_sf<true, true, true>(jobs, o3, cnt[3], graphs, preps, smem[1], s);
  } else {
    launch_sf<false, false, false>(jobs, order, cnt[0], graphs, preps, smem[0], s);
    launch_sf<true, false, false>(jobs, o1, cnt[1], graphs, preps, smem[0], s);
    launch_sf<false, false, true>(jobs, o2, cnt[2], graphs, preps, smem[1], s);
    launch_sf<true, false, true>(jobs, o3, cnt[3], graphs, preps, smem[1], s);
  }
}

}  // namespace bx

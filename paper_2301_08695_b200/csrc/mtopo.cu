// m-TOPO (place_mtopo, proj/src/placers.cpp:314-365) as one CTA per job.
//
// 1. Min-index Kahn order (meta_topo_order, transforms.cpp:446-479) in
//    bursts. Let U be the smallest unpopped node. Every node below U is
//    popped, so the smallest ready node is the first ready node >= U. Call a
//    node BLOCKED while some parent with a LARGER index is unpopped, and let
//    B be the first blocked node >= U. Every unpopped node y in [U, B) is
//    ready at its turn when the pops go U, U+1, ...: its parents below U are
//    popped, those in [U, y) are popped just before it, and it has no
//    unpopped parent above it. Nodes made ready by these pops are >= U and
//    not below the next node of the run, so the min-index order pops exactly
//    the unpopped nodes of [U, B) in ascending order — one parallel step
//    (ranks by popcount over the popped bitset). When U itself is blocked,
//    the next pop is the first ready node >= U (a bitset search), popped
//    alone. A graph whose edges all go from smaller to larger index (every
//    model-shaped graph here) is one burst: the identity order.
// 2. Balanced fill (placers.cpp:337-347): with non-negative needs the greedy
//    "next device once used + need > cap" puts boundary d+1 at the first x
//    after boundary d with S[x] - S[boundary d - 1] > cap, S the inclusive
//    prefix sum of needs in topo order: a block scan plus one binary search
//    per device. (Any negative need: the greedy replayed by one thread.)
// 3. Schedule estimate (placers.cpp:350-362), parallel comm: devices are
//    contiguous topo chunks and parents precede children, so device d
//    depends only on devices < d; a remote parent's tensor lands at its
//    finish + c of the edge to its FIRST consumer on d in topo order (later
//    consumers hit the cache entry). Per device, 1 node per thread: the
//    data-ready time A_l, then a block max-plus scan
//    f_l = max(f_{l-1} + k_l, A_l + k_l). Sequential comm keeps the
//    reference fold (queue tails) on one thread.
#include <algorithm>

#include "sched_common.cuh"

namespace bx {

constexpr int kTopoThreads = 512;
constexpr int kTopoWarps = kTopoThreads / 32;
constexpr int kTopoBig = 1 << 30;  // pend[] of a popped node is pushed below -kTopoBig / 2

struct TopoShared {
  int wmin[2][kTopoWarps];
  long long wsum[2][kTopoWarps];
  long long wa[2][kTopoWarps], wb[2][kTopoWarps];
  int bound[2];
};

// Block-wide minimum; one barrier. `par` alternates the scratch row so the
// next call never overwrites a row another thread may still be reading.
__device__ __forceinline__ int block_min(TopoShared &S, int &par, int v) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  v = static_cast<int>(__reduce_min_sync(kFull, static_cast<unsigned>(v)));
  if (lane == 0) S.wmin[par][warp] = v;
  __syncthreads();
  int r = lane < kTopoWarps ? S.wmin[par][lane] : INT32_MAX;
  par ^= 1;
  return static_cast<int>(__reduce_min_sync(kFull, static_cast<unsigned>(r)));
}

// Block-wide exclusive prefix sum of v (int64), and the block total.
__device__ __forceinline__ long long block_scan(TopoShared &S, int &par, long long v, long long &total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long t = __shfl_up_sync(kFull, inc, o);
    if (lane >= o) inc += t;
  }
  if (lane == 31) S.wsum[par][warp] = inc;
  __syncthreads();
  long long before = 0, tot = 0;
  for (int w = 0; w < kTopoWarps; ++w) {
    const long long x = S.wsum[par][w];
    if (w < warp) before += x;
    tot += x;
  }
  par ^= 1;
  total = tot;
  return before + inc - v;
}

// Block-wide inclusive max-plus scan of (a, b) pairs: composing (a1, b1)
// then (a2, b2) gives (a1 + a2, max(b1 + a2, b2)); returns the inclusive
// pair and the block total.
__device__ __forceinline__ void block_maxplus(TopoShared &S, int &par, long long &a, long long &b, long long &ta,
                                              long long &tb) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long a2 = __shfl_up_sync(kFull, a, o), b2 = __shfl_up_sync(kFull, b, o);
    if (lane >= o) {
      b = max64(b2 + a, b);
      a = a2 + a;
    }
  }
  if (lane == 31) {
    S.wa[par][warp] = a;
    S.wb[par][warp] = b;
  }
  __syncthreads();
  long long pa = 0, pb = INT64_MIN / 4, qa = 0, qb = INT64_MIN / 4;  // prefix of lower warps; block total
  for (int w = 0; w < kTopoWarps; ++w) {
    const long long wa = S.wa[par][w], wb = S.wb[par][w];
    if (w < warp) {
      pb = max64(pb + wa, wb);
      pa = pa + wa;
    }
    qb = max64(qb + wa, wb);
    qa = qa + wa;
  }
  par ^= 1;
  b = max64(pb + a, b);
  a = pa + a;
  ta = qa;
  tb = qb;
}

// First index >= from whose bit is set, or V.
__device__ __forceinline__ int block_ffs(TopoShared &S, int &par, const uint32_t *bits, int from, int V) {
  const int nw = (V + 31) >> 5;
  for (int w0 = from >> 5; w0 < nw; w0 += kTopoThreads) {
    const int w = w0 + static_cast<int>(threadIdx.x);
    int cand = INT32_MAX;
    if (w < nw) {
      uint32_t word = bits[w];
      if (w == (from >> 5)) word &= ~0u << (from & 31);
      if (word) cand = 32 * w + __ffs(word) - 1;
    }
    const int r = block_min(S, par, cand);
    if (r != INT32_MAX) return r < V ? r : V;
  }
  return V;
}

// Children of a just-popped node y: pending counts, the ready bit when the
// last parent lands, the blocked bit when the last larger-index parent does.
__device__ __forceinline__ void topo_release(const DGraph &g, int y, int *pend, int *pbwd, uint32_t *ready,
                                             uint32_t *blocked) {
  for (int e = g.out_off[y]; e < g.out_off[y + 1]; ++e) {
    const int c = g.edst[e];
    if (atomicSub(pend + c, 1) == 1) atomicOr(ready + (c >> 5), 1u << (c & 31));
    if (y > c && atomicSub(pbwd + c, 1) == 1) atomicAnd(blocked + (c >> 5), ~(1u << (c & 31)));
  }
}

__global__ void __launch_bounds__(kTopoThreads) k_place_topo_cta(const DJob *jobs, const DGraph *graphs,
                                                                 const DPrep *preps, int smem_words) {
  extern __shared__ __align__(16) uint32_t tsm[];
  __shared__ TopoShared S;
  __shared__ long long s_cap;
  __shared__ int s_neg;
  const int tid = threadIdx.x;
  const DJob jb = jobs[blockIdx.x];
  if (jb.skip || jb.algo != 0) return;
  const DGraph g = graphs[jb.graph];
  const DPrep pr = preps[jb.prep];
  const int V = g.V, n = jb.n;
  int par = 0;
  long long t_mark = clock64();
  // profile builds (plan option profile): SM cycles per phase into jb.prof
  // (0 warm + cap, 1 order, 2 fill, 3 devices, 4 estimate)
#define TMARK(k)                                   \
  do {                                             \
    if (jb.prof && tid == 0) {                     \
      const long long now_ = clock64();            \
      jb.prof[k] = now_ - t_mark;                  \
      t_mark = now_;                               \
    }                                              \
  } while (0)
  // pull the graph arrays the dependent chains below walk (in-CSR, out-CSR,
  // comm times, needs, compute times) into this SM's L1 first: independent
  // 16-byte loads, one per 32-byte sector
  if (static_cast<size_t>(V) * 64 + static_cast<size_t>(g.E) * 20 <= 160 * 1024) {
    unsigned acc = 0;
    auto warm = [&](const void *ptr, size_t bytes) {
      const uintptr_t a0 = reinterpret_cast<uintptr_t>(ptr) & ~uintptr_t(31);
      const uintptr_t a1 = reinterpret_cast<uintptr_t>(ptr) + bytes;
      for (uintptr_t q = a0 + 32 * static_cast<uintptr_t>(tid); q < a1; q += 32 * kTopoThreads)
        acc ^= __ldg(reinterpret_cast<const unsigned *>(q));
    };
    warm(g.in_off, 4 * size_t(V + 1));
    warm(g.in_src, 4 * size_t(g.E));
    warm(g.out_off, 4 * size_t(V + 1));
    warm(g.edst, 4 * size_t(g.E));
    warm(g.inpos, 4 * size_t(g.E));
    warm(pr.in_c, 8 * size_t(g.E));
    warm(g.need, 8 * size_t(V));
    warm(g.k, 8 * size_t(V));
    asm volatile("" ::"r"(acc));
  }
  // cap = ceil(total / n) + largest (largest starts at 0); infeasible comes
  // before the acyclicity check
  if (tid == 0) s_cap = 0;
  {
    long long total = 0, largest = 0;
    int neg = 0;
    for (int j = tid; j < V; j += kTopoThreads) {
      const int64_t b = g.need[j];
      total += b;
      largest = max64(largest, b);
      neg |= b < 0;
    }
    long long tot;
    block_scan(S, par, total, tot);  // its barrier also orders s_cap's reset
    for (int o = 16; o > 0; o >>= 1) largest = max64(largest, __shfl_xor_sync(kFull, largest, o));
    if ((tid & 31) == 0) atomicMax(&s_cap, largest);
    neg = __syncthreads_or(neg);
    int64_t mincap = jb.cap[0];
    for (int d = 1; d < n; ++d) mincap = min64(mincap, jb.cap[d]);
    const int64_t cap = (tot + n - 1) / n + s_cap;
    __syncthreads();
    if (cap > mincap) {
      if (tid == 0) set_err(jb.err, kInfeasible, E_TOPO_CAP, cap, mincap);
      return;
    }
    if (tid == 0) {
      s_cap = cap;
      s_neg = neg;
    }
  }
  if (g.flags[0] != V) {
    if (tid == 0) set_err(jb.err, kValidation, E_CYCLE, 0, 0);
    return;
  }
  if (g.flags[1]) {  // a negative tensor size: comm_time throws (cost_model.cpp:31-33), as in the list placers
    if (tid == 0) set_err(jb.err, kValidation, E_NEG_BYTES, 0, 0);
    return;
  }
  __syncthreads();
  const int64_t cap = s_cap;
  const bool neg_need = s_neg != 0;

  TMARK(0);
  // ---- 1. min-index Kahn in bursts --------------------------------------------
  int32_t *order = jb.exec_order;  // the topo order doubles as the exec lists
  int any_bwd = 0;
  for (int y = tid; y < V; y += kTopoThreads) {
    const int e = g.in_off[y + 1];
    any_bwd |= e > g.in_off[y] && g.in_src[e - 1] > y;  // in_src ascending: the last parent is the largest
  }
  const bool ident = !__syncthreads_or(any_bwd);
  if (ident) {
    // numbered topologically: one burst over [0, V), the identity
    for (int x = tid; x < V; x += kTopoThreads) order[x] = x;
  } else {
    const int nw = (V + 31) >> 5;
    uint32_t *popped, *ready, *blocked;
    int *pend, *pbwd;
    {
      // bitsets (and, when they fit too, the counters) in shared memory;
      // otherwise in the job's byte scratch (V * n >= 3 V / 8 bytes) and its
      // int32 arrays
      const bool bits_sm = 3 * nw <= smem_words;
      const bool cnt_sm = bits_sm && 3 * nw + 2 * V <= smem_words;
      uint32_t *bb = bits_sm ? tsm : reinterpret_cast<uint32_t *>(jb.dead);
      popped = bb;
      ready = bb + nw;
      blocked = bb + 2 * nw;
      pend = cnt_sm ? reinterpret_cast<int *>(tsm + 3 * nw) : jb.pending;
      pbwd = cnt_sm ? reinterpret_cast<int *>(tsm + 3 * nw + V) : jb.alive;
    }
    for (int w = tid; w < nw; w += kTopoThreads) {
      popped[w] = 0;
      ready[w] = 0;
      blocked[w] = 0;
    }
    __syncthreads();
    for (int y = tid; y < V; y += kTopoThreads) {
      const int b = g.in_off[y], e = g.in_off[y + 1];
      int bw = 0;
      for (int x = e - 1; x >= b && g.in_src[x] > y; --x) ++bw;  // in_src ascending
      pend[y] = e - b;
      pbwd[y] = bw;
      if (e == b) atomicOr(ready + (y >> 5), 1u << (y & 31));
      if (bw) atomicOr(blocked + (y >> 5), 1u << (y & 31));
    }
    __syncthreads();
    int cnt = 0, U = 0;
    while (cnt < V) {
      // U = first unpopped: scan the complement of `popped` word by word
      {
        int w0 = U >> 5;
        int found = V;
        for (; w0 < nw; w0 += kTopoThreads) {
          const int w = w0 + tid;
          int cand = INT32_MAX;
          if (w < nw) {
            uint32_t word = ~popped[w];
            if (w == (U >> 5)) word &= ~0u << (U & 31);
            if (word) cand = 32 * w + __ffs(word) - 1;
          }
          const int r = block_min(S, par, cand);
          if (r != INT32_MAX) {
            found = r < V ? r : V;
            break;
          }
        }
        U = found;
      }
      if (U >= V) break;
      const int B = block_ffs(S, par, blocked, U, V);
      if (B > U) {
        // burst: the unpopped nodes of [U, B) in ascending order; one word per thread
        const int wb = U >> 5, we = (B - 1) >> 5;
        const int cnt0 = cnt;
        for (int w0 = wb; w0 <= we; w0 += kTopoThreads) {
          const int w = w0 + tid;
          uint32_t take = 0;
          if (w <= we) {
            uint32_t m = ~popped[w];
            if (w == wb) m &= ~0u << (U & 31);
            if (w == we && ((B & 31) != 0)) m &= (1u << (B & 31)) - 1u;
            take = m;
          }
          long long tot;
          const int pos = cnt + static_cast<int>(block_scan(S, par, __popc(take), tot));
          if (take) {
            uint32_t m = take;
            int k = pos;
            while (m) {
              const int b = __ffs(m) - 1;
              m &= m - 1;
              const int y = 32 * w + b;
              order[k++] = y;
              pend[y] = -kTopoBig;
            }
            popped[w] |= take;
            ready[w] &= ~take;
          }
          cnt += static_cast<int>(tot);
        }
        __syncthreads();
        for (int x = cnt0 + tid; x < cnt; x += kTopoThreads) topo_release(g, order[x], pend, pbwd, ready, blocked);
        __syncthreads();
        U = B;
      } else {
        // U is blocked: the first ready node >= U pops alone
        const int r = block_ffs(S, par, ready, U, V);
        if (tid == 0) {
          order[cnt] = r;
          pend[r] = -kTopoBig;
          popped[r >> 5] |= 1u << (r & 31);
          ready[r >> 5] &= ~(1u << (r & 31));
        }
        ++cnt;
        __syncthreads();
        for (int e = g.out_off[r] + tid; e < g.out_off[r + 1]; e += kTopoThreads) {
          const int c = g.edst[e];
          if (atomicSub(pend + c, 1) == 1) atomicOr(ready + (c >> 5), 1u << (c & 31));
          if (r > c && atomicSub(pbwd + c, 1) == 1) atomicAnd(blocked + (c >> 5), ~(1u << (c & 31)));
        }
        __syncthreads();
      }
    }

  }  // bursts
  __syncthreads();

  TMARK(1);
  // ---- 2. balanced fill; the last device absorbs the rest --------------------------
  int64_t *S_need = jb.urgent;  // inclusive prefix sums of needs in topo order
  {
    long long carry = 0;
    for (int x0 = 0; x0 < V; x0 += kTopoThreads) {
      const int x = x0 + tid;
      const long long b = x < V ? g.need[order[x]] : 0;
      long long tot;
      const long long ex = block_scan(S, par, b, tot);
      if (x < V) S_need[x] = carry + ex + b;
      carry += tot;
    }
  }
  __syncthreads();
  int32_t *off = jb.exec_off;
  if (tid < 32) {
    const int lane = tid;
    int d = 0;
    if (!neg_need) {
      // boundary d+1 = first x > s_d (x >= 0 for d = 0) with S[x] - S[s_d - 1] > cap
      // (S non-decreasing): a 32-way search per device, 32 probes per step
      int s = 0;
      for (; d + 1 < n; ++d) {
        const long long base = s > 0 ? S_need[s - 1] : 0;
        int lo = d == 0 ? 0 : s + 1, hi = V;  // first true in [lo, hi); hi = V: none
        while (lo < hi) {
          const int step = (hi - lo + 31) / 32;
          const int x = lo + lane * step;
          const bool pr = x < hi && S_need[x] - base > cap;
          const unsigned m = __ballot_sync(kFull, pr);
          if (step == 1) {
            lo = hi = m ? lo + __ffs(m) - 1 : hi;
          } else if (!m) {
            lo += ((hi - 1 - lo) / step) * step + 1;  // past the last probe below hi
          } else {
            const int f = __ffs(m) - 1;
            if (f == 0) {
              hi = lo;  // x_0 = lo is the first
            } else {
              hi = lo + f * step + 1;  // the answer is in (x_{f-1}, x_f]
              lo = lo + (f - 1) * step + 1;
            }
          }
        }
        if (lo >= V) break;
        if (lane == 0) off[d + 1] = lo;
        s = lo;
      }
    } else if (lane == 0) {
      long long used = 0;
      for (int x = 0; x < V; ++x) {
        const long long b = g.need[order[x]];
        if (used + b > cap && d + 1 < n) {
          off[++d] = x;
          used = 0;
        }
        used += b;
      }
    }
    d = __shfl_sync(kFull, d, 0);
    if (lane == 0) {
      off[0] = 0;
      for (int e = d + 1; e <= n; ++e) off[e] = V;
    }
  }
  __syncthreads();
  TMARK(2);
  int32_t *tpos = jb.rpos;
  // identity order, parallel comm, small graph: finish times and devices in
  // shared memory for the estimate (the bitsets are not needed)
  const bool fast = ident && jb.mode == 1 && static_cast<size_t>(V) * 18 + 16 <= static_cast<size_t>(smem_words) * 4;
  long long *fin_s = reinterpret_cast<long long *>(tsm);
  long long *A_s = fin_s + V;
  uint16_t *dev_s = reinterpret_cast<uint16_t *>(A_s + V);
  for (int x = tid; x < V; x += kTopoThreads) {
    int d = 0;
    while (off[d + 1] <= x) ++d;  // n is small; the rosters' largest chunk count
    const int j = order[x];
    jb.device_of[j] = d;
    tpos[j] = x;
    if (fast) dev_s[j] = static_cast<uint16_t>(d);
  }
  __syncthreads();

  TMARK(3);
  if (fast) {
    // ---- 3. schedule estimate, parallel comm, identity order: node index =
    // topo position, so a remote parent's first consumer on device d is its
    // first out-edge (ascending dst) at or past off[d]. Per device: the
    // arrival terms edge-parallel over the device's in-edges (its nodes are
    // contiguous, so are their in-CSR slots) into A_s, then the block scans.
    for (int x = tid; x < V; x += kTopoThreads) A_s[x] = 0;
    __syncthreads();
    for (int d = 0; d < n; ++d) {
      const int o = off[d], len = off[d + 1] - o;
      const int xb = g.in_off[o], xe = g.in_off[o + len];
      for (int x = xb + tid; x < xe; x += kTopoThreads) {
        const int i = g.in_src[x];
        if (dev_s[i] == d) continue;  // earlier on this device: covered by the chain
        int lo = g.out_off[i], hi = g.out_off[i + 1];  // first out-edge with dst >= o
        while (lo < hi) {
          const int mid = (lo + hi) >> 1;
          if (g.edst[mid] < o) lo = mid + 1;
          else hi = mid;
        }
        // the consumer: the in-CSR slot's node (binary search on in_off is
        // avoided: x's node is the one whose in-CSR range holds x)
        atomicMax(reinterpret_cast<long long *>(A_s) + g.edst[g.in_edge[x]], fin_s[i] + pr.in_c[g.inpos[lo]]);
      }
      __syncthreads();
      long long prev = 0;
      for (int b0 = 0; b0 < len; b0 += kTopoThreads) {
        const int idx = b0 + tid;
        const int j = o + idx;
        const long long kk = idx < len ? g.k[j] : 0, A = idx < len ? A_s[j] : 0;
        long long a = kk, bb = A + kk, ta, tb;
        block_maxplus(S, par, a, bb, ta, tb);
        const long long f = max64(prev + a, bb);
        if (idx < len) {
          jb.start[j] = f - kk;
          fin_s[j] = f;
        }
        prev = max64(prev + ta, tb);
      }
      __syncthreads();  // device d's finishes before device d + 1 reads them
    }
    TMARK(4);
    if (tid == 0) {
      jb.stats[0] = jb.stats[1] = jb.stats[2] = 0;
      set_err(jb.err, kOk, E_NONE, 0, 0);
    }
    return;
  }
  if (jb.mode == 1) {
    // ---- 3. schedule estimate, parallel comm --------------------------------------
    for (int y = tid; y < g.E; y += kTopoThreads) {  // y = edge id = out-CSR slot
      const int i = g.esrc[y], j = g.edst[y], pj = jb.device_of[j];
      if (jb.device_of[i] != pj) jb.cache[static_cast<int64_t>(i) * n + pj] = INT64_MAX;
    }
    __syncthreads();
    for (int y = tid; y < g.E; y += kTopoThreads) {
      const int i = g.esrc[y], j = g.edst[y], pj = jb.device_of[j];
      if (jb.device_of[i] != pj)
        atomicMin(reinterpret_cast<long long *>(jb.cache + static_cast<int64_t>(i) * n + pj),
                  (static_cast<long long>(tpos[j]) << 32) | g.inpos[y]);
    }
    __syncthreads();
    for (int d = 0; d < n; ++d) {
      const int o = off[d], len = off[d + 1] - o;
      long long prev = 0;
      for (int b0 = 0; b0 < len; b0 += kTopoThreads) {
        const int idx = b0 + tid;
        long long A = 0, kk = 0;
        int j = -1;
        if (idx < len) {
          j = order[o + idx];
          kk = g.k[j];
          for (int x = g.in_off[j]; x < g.in_off[j + 1]; ++x) {
            const int i = g.in_src[x];
            if (jb.device_of[i] == d) continue;  // earlier on this device: covered by the chain
            const int first = static_cast<int>(jb.cache[static_cast<int64_t>(i) * n + d] & 0xffffffffll);
            A = max64(A, jb.finish[i] + pr.in_c[first]);
          }
        }
        long long a = kk, bb = A + kk, ta, tb;
        block_maxplus(S, par, a, bb, ta, tb);
        const long long f = max64(prev + a, bb);
        if (idx < len) {
          jb.start[j] = f - kk;
          jb.finish[j] = f;
        }
        prev = max64(prev + ta, tb);
      }
      __syncthreads();  // device d's finishes before device d + 1 reads them
    }
    if (tid == 0) {
      jb.stats[0] = jb.stats[1] = jb.stats[2] = 0;
      set_err(jb.err, kOk, E_NONE, 0, 0);
    }
    return;
  }
  if (tid == 0) {
    // schedule estimate (placers.cpp:350-362), sequential comm: the queue
    // tails make it a fold in topo order; every device_of is set before it
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
    c.F = jb.sc_val;
    c.tail = jb.sc_val + n;
    for (int d = 0; d < n; ++d) c.F[d] = c.tail[d] = 0;
    for (int x = 0; x < V; ++x) {
      const int j = order[x];
      const int p = jb.device_of[j];
      int cn;
      const int64_t t = commit_fold(c, j, p, &cn);
      jb.start[j] = t;
      jb.finish[j] = t + g.k[j];
      c.F[p] = jb.finish[j];
    }
    jb.stats[0] = jb.stats[1] = jb.stats[2] = 0;
    set_err(jb.err, kOk, E_NONE, 0, 0);
  }
}

#undef TMARK

// Acyclicity (meta_topo_order's CycleError, transforms.cpp:446-479): the set
// of nodes Kahn's algorithm cannot peel does not depend on the pop order, so
// any peel order finds the same residue. One CTA per graph.
//
// Sweeps (warp 0): walk the nodes in index order, 32 at a time, and peel
// every node whose parents are all peeled — earlier in this sweep or before.
// A parent with a larger index must have been peeled by an earlier sweep;
// parents inside the 32-node chunk resolve by a ballot fixpoint (the chunk's
// edges go forward, so it converges). A graph numbered topologically peels
// in one sweep whatever its depth (a level-synchronous peel pays a CTA
// barrier per level: 1.25 ms on C1's 3.6k-group chain); each further sweep
// follows one more backward edge along a path. When sweeps stop paying
// (more than kAcycSweeps), the CTA finishes with a level-synchronous peel
// over the remaining nodes' pending counts.
// Scratch: the peeled bitset in shared memory (over `iota`, free once the
// need sort has run, past 393k nodes); queue[0, 2V) for the level peel;
// indeg_left ends > 0 exactly on the residue (the cycle message reads it).
constexpr int kAcycSmemWords = 12000;
constexpr int kAcycSweeps = 8;
__global__ void __launch_bounds__(kTopoThreads) k_acyclic(DGraph *graphs, int32_t *const *queues) {
  __shared__ uint32_t bsm[kAcycSmemWords];
  __shared__ int s_cnt[3], s_peeled;
  DGraph g = graphs[blockIdx.x];
  int32_t *q = queues[blockIdx.x];
  const int tid = threadIdx.x, lane = tid & 31, V = g.V;
  const int nw = (V + 31) >> 5;
  uint32_t *done = nw <= kAcycSmemWords ? bsm : reinterpret_cast<uint32_t *>(g.iota);
  // no edge from a larger to a smaller index: the numbering is a topological
  // order, nothing to peel (every model-shaped graph here); the pass also
  // pulls the in-CSR into L1 for warp 0's sweeps otherwise
  int bwd = 0;
  for (int y = tid; y < V; y += kTopoThreads) {
    const int e = g.in_off[y + 1];
    bwd |= e > g.in_off[y] && g.in_src[e - 1] > y;  // in_src ascending: the last parent is the largest
  }
  if (!__syncthreads_or(bwd)) {
    for (int y = tid; y < V; y += kTopoThreads) g.indeg_left[y] = 0;
    if (tid == 0) g.flags[0] = V;
    return;
  }
  for (int w = tid; w < nw; w += kTopoThreads) done[w] = 0;
  __syncthreads();
  if (tid < 32) {
    int peeled = 0, first = 0;  // first: chunk holding the smallest unpeeled node
    for (int sweep = 0; sweep < kAcycSweeps && peeled < V; ++sweep) {
      int got = 0, nfirst = -1;
      for (int c = first; c < nw; ++c) {
        const int y = 32 * c + lane;
        const uint32_t dw = done[c];
        bool cand = false;
        uint32_t inm = 0;
        if (y < V && !((dw >> lane) & 1u)) {
          cand = true;
          for (int x = g.in_off[y]; x < g.in_off[y + 1] && cand; ++x) {
            const int p = g.in_src[x];
            if (p >= 32 * c && p < y) {
              inm |= 1u << (p - 32 * c);  // same chunk: resolved below
            } else if (!((done[p >> 5] >> (p & 31)) & 1u)) {
              cand = false;  // an unpeeled parent outside the chunk (later, or earlier and stuck)
            }
          }
        }
        unsigned T = __ballot_sync(kFull, cand);
        while (true) {
          const unsigned T2 = __ballot_sync(kFull, cand && (inm & ~T) == 0u);
          if (T2 == T) break;
          T = T2;
        }
        __syncwarp();  // every lane has read done[c] and its parents' words
        if (lane == 0 && T) done[c] = dw | T;
        __syncwarp();
        got += __popc(T);
        if (nfirst < 0 && (dw | T) != (y - lane + 32 <= V ? 0xffffffffu : (1u << (V & 31)) - 1u)) nfirst = c;
      }
      peeled += got;
      first = nfirst < 0 ? nw : nfirst;
      if (got == 0) break;
    }
    if (lane == 0) s_peeled = peeled;
  }
  __syncthreads();
  int peeled = s_peeled;
  if (peeled < V) {
    // level-synchronous peel of the rest: pending = unpeeled parents
    int *pend = g.indeg_left;
    if (tid == 0) s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
    __syncthreads();
    for (int y = tid; y < V; y += kTopoThreads) {
      int left = 0;
      if (!((done[y >> 5] >> (y & 31)) & 1u)) {
        for (int x = g.in_off[y]; x < g.in_off[y + 1]; ++x) {
          const int p = g.in_src[x];
          left += !((done[p >> 5] >> (p & 31)) & 1u);
        }
        if (left == 0) q[atomicAdd(&s_cnt[0], 1)] = y;
      }
      pend[y] = left;
    }
    __syncthreads();
    for (int L = 0;; ++L) {
      const int cnt = s_cnt[L % 3];
      if (cnt == 0) break;
      const int32_t *in = q + ((L & 1) ? V : 0);
      int32_t *out = q + ((L & 1) ? 0 : V);
      int *next = &s_cnt[(L + 1) % 3];
      if (tid == 0) s_cnt[(L + 2) % 3] = 0;
      peeled += cnt;
      for (int x = tid; x < cnt; x += kTopoThreads) {
        const int u = in[x];
        for (int y = g.out_off[u]; y < g.out_off[u + 1]; ++y) {
          const int v = g.edst[y];
          if (atomicSub(&pend[v], 1) == 1) out[atomicAdd(next, 1)] = v;
        }
      }
      __syncthreads();
    }
  } else {
    for (int y = tid; y < V; y += kTopoThreads) g.indeg_left[y] = 0;
  }
  if (tid == 0) g.flags[0] = peeled;
}

void launch_kahn(DGraph *graphs_dev, int32_t *const *queues_dev, int ngraphs, cudaStream_t s) {
  if (ngraphs > 0) k_acyclic<<<ngraphs, kTopoThreads, 0, s>>>(graphs_dev, queues_dev);
}

// One CTA per job of the plan (list jobs exit at once); shared memory holds
// the bitsets and counters of graphs up to smem_bytes.
void launch_topo(const DJob *jobs, int njobs, const DGraph *graphs, const DPrep *preps, size_t smem_bytes,
                 cudaStream_t s) {
  if (njobs <= 0) return;
  cudaFuncSetAttribute(k_place_topo_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem_bytes));
  k_place_topo_cta<<<njobs, kTopoThreads, smem_bytes, s>>>(jobs, graphs, preps, static_cast<int>(smem_bytes / 4));
}

// Shared memory for a graph of V nodes: bitsets plus counters when they fit
// under `limit` bytes, else bitsets only (counters in HBM), else none.
size_t topo_smem_bytes(int V, size_t limit) {
  const size_t nw = (static_cast<size_t>(V) + 31) / 32;
  // bitsets + counters, or (identity order) finish times + devices
  const size_t full = std::max(4 * (3 * nw + 2 * static_cast<size_t>(V)), 18 * static_cast<size_t>(V) + 16);
  if (full <= limit) return (full + 15) & ~size_t(15);
  return 12 * nw <= limit ? 12 * nw : 0;
}

}  // namespace bx

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

#include "sched_common.cuh"

namespace bx {


// ---------------------------------------------------------------- K1 ----
// Per (graph, comm model): in-CSR gather of src + comm_time per slot, and
// c_max. Bytes per edge: 4 (in_edge) + 4 (esrc) + 8 (ebytes) read, 4 + 8
// written.
__device__ __forceinline__ void prep_edges(const DGraph &g, const DPrep &pr, int write_src, int tid, int nthreads) {
  int64_t best = 0;
  int neg = 0;
  for (int x = tid; x < g.E; x += nthreads) {
    int e = g.in_edge[x];
    int64_t b = g.ebytes[e];
    if (b < 0) {
      neg = 1;
      b = 0;
    }
    if (write_src) {
      g.in_src[x] = g.esrc[e];
      g.inpos[e] = x;
    }
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

// need[j] = perm + out + temp (reserve_bytes, placers.hpp:43-45); the sum of
// compute times and a negative-time flag (the small-frontier kernel's bounds).
__device__ __forceinline__ void prep_nodes(const DGraph &g, int tid, int nthreads) {
  unsigned long long ks = 0;
  int neg = 0;
  for (int j = tid; j < g.V; j += nthreads) {
    int64_t v = g.perm[j] + g.outb[j] + g.temp[j];
    g.need[j] = v;
    g.iota[j] = j;
    g.indeg_left[j] = g.in_off[j + 1] - g.in_off[j];
    const int64_t k = g.k[j];
    if (k < 0) neg = 1;
    else ks += static_cast<unsigned long long>(k);
  }
  for (int o = 16; o > 0; o >>= 1) {
    ks += __shfl_xor_sync(kFull, ks, o);
    neg |= __shfl_xor_sync(kFull, neg, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (ks) atomicAdd(reinterpret_cast<unsigned long long *>(g.ksum), ks);
    if (neg) atomicOr(&g.flags[2], 1);
  }
}

// Every prepared (graph, comm model) of a plan in one launch: blockIdx.y is
// the prep; the first prep of each graph also derives the graph-level node
// arrays and the in-CSR source gather.
__global__ void k_prep_all(const DGraph *graphs, const DPrep *preps) {
  const DPrep pr = preps[blockIdx.y];
  const DGraph g = graphs[pr.graph];
  const int tid = blockIdx.x * blockDim.x + threadIdx.x, nth = gridDim.x * blockDim.x;
  prep_edges(g, pr, pr.first, tid, nth);
  if (pr.first) prep_nodes(g, tid, nth);
}

// Per-step zero / 0xff fills of a plan's workspace (key caches, dead flags,
// error records, output offsets, ...) in one launch instead of one memset per
// array: the host splits every fill into chunks of at most kFillChunk bytes
// (chunk starts stay 16-byte aligned), each CTA stores its chunks with 16-byte
// vector stores.
__global__ void __launch_bounds__(256) k_fill(const FillChunk *__restrict__ t, int n) {
  for (int c = blockIdx.x; c < n; c += gridDim.x) {
    const FillChunk f = t[c];
    unsigned char *p = reinterpret_cast<unsigned char *>(f.ptr);
    const unsigned w = f.word;
    const uint4 w4 = make_uint4(w, w, w, w);
    // chunk starts are 4-byte aligned, so the 16-byte-aligned body starts on a word boundary
    const size_t head = (16 - (reinterpret_cast<uintptr_t>(p) & 15)) & 15;
    const size_t pre = head < f.bytes ? head : f.bytes;
    for (size_t i = threadIdx.x; i < pre; i += blockDim.x) p[i] = static_cast<unsigned char>(w >> (8 * (i & 3)));
    const size_t body = (f.bytes - pre) >> 4;
    uint4 *q = reinterpret_cast<uint4 *>(p + pre);
    for (size_t i = threadIdx.x; i < body; i += blockDim.x) q[i] = w4;
    for (size_t i = pre + (body << 4) + threadIdx.x; i < f.bytes; i += blockDim.x)
      p[i] = static_cast<unsigned char>(w >> (8 * (i & 3)));
  }
}

// Acyclicity (meta_topo_order's CycleError, transforms.cpp:446-479): the set
// of nodes Kahn's algorithm cannot peel does not depend on the pop order,
// so a level-synchronous peel finds the same residue. One CTA per graph;
// the frontier ping-pongs through `queue` (2*V ints of scratch).
__global__ void k_kahn(DGraph *graphs, int32_t *const *queues) {
  // level-synchronous peel, one barrier per level: level L reads queue buffer
  // L%2 with count s_n[L%3], appends to buffer (L+1)%2 / s_n[(L+1)%3], and
  // clears s_n[(L+2)%3] (last read at level L-1, next written at level L+1)
  DGraph g = graphs[blockIdx.x];
  int32_t *q = queues[blockIdx.x];
  __shared__ int s_n[3];
  __shared__ int s_total;
  const int V = g.V;
  if (threadIdx.x == 0) {
    s_n[0] = s_n[1] = s_n[2] = 0;
    s_total = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    if (g.indeg_left[j] == 0) q[atomicAdd(&s_n[0], 1)] = j;
  }
  __syncthreads();
  for (int L = 0;; ++L) {
    const int cnt = s_n[L % 3];
    if (cnt == 0) break;
    const int32_t *in = q + ((L & 1) ? V : 0);
    int32_t *out = q + ((L & 1) ? 0 : V);
    int *next = &s_n[(L + 1) % 3];
    if (threadIdx.x == 0) {
      s_total += cnt;
      s_n[(L + 2) % 3] = 0;
    }
    for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
      const int u = in[x];
      for (int y = g.out_off[u]; y < g.out_off[u + 1]; ++y) {
        const int v = g.edst[y];
        if (atomicSub(&g.indeg_left[v], 1) == 1) out[atomicAdd(next, 1)] = v;
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) g.flags[0] = s_total;
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
  if (g.flags[1]) {  // a negative tensor size: comm_time throws (cost_model.cpp:31-33), as in the list placers
    if (lane == 0) set_err(jb.err, kValidation, E_NEG_BYTES, 0, 0);
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
    // one REDUX for the minimum node; its lane (ids are unique) moves the
    // last ready slot into the hole
    const int mine = best;
    best = static_cast<int>(__reduce_min_sync(kFull, static_cast<unsigned>(best)));
    if (mine == best) {
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
  {
    // balanced fill; the last device absorbs the rest (placers.cpp:337-347).
    // The greedy is sequential, but its inputs are not: the warp loads 32
    // nodes' needs at once and every lane replays the same greedy over them
    // from registers, keeping the device of its own node.
    int dev = 0;
    int64_t used = 0;
    if (lane == 0) jb.exec_off[0] = 0;
    for (int base = 0; base < V; base += 32) {
      const int x = base + lane;
      const int j = x < V ? order[x] : 0;
      const int64_t b = x < V ? g.need[j] : 0;
      const int cntb = V - base < 32 ? V - base : 32;
      int mine = 0;
      for (int l = 0; l < cntb; ++l) {
        const int64_t bl = __shfl_sync(kFull, b, l);
        if (used + bl > cap && dev + 1 < n) {
          if (lane == 0) jb.exec_off[dev + 1] = base + l;
          ++dev;
          used = 0;
        }
        if (l == lane) mine = dev;
        used += bl;
      }
      if (x < V) jb.device_of[j] = mine;
    }
    if (lane == 0)
      for (int d = dev + 1; d <= n; ++d) jb.exec_off[d] = V;
  }
  __syncwarp();
  if (c.mode == 1) {
    // schedule estimate, parallel comm (placers.cpp:350-362), warp-parallel:
    // a remote parent's tensor lands on p at finish + c_e of the edge to its
    // FIRST consumer on p in topo order (later consumers hit that cache
    // entry), and every parent precedes its child in topo order, so device d
    // (a contiguous topo chunk) depends only on devices < d and on its own
    // predecessor: walk the devices in order, 32 nodes at a time, with a
    // max-plus scan f_l = max(f_{l-1} + k_l, A_l + k_l).
    int32_t *tpos = jb.pending;  // free after Kahn
    for (int x = lane; x < V; x += 32) tpos[order[x]] = x;
    __syncwarp();
    for (int y = lane; y < g.E; y += 32) {  // y = edge id = out-CSR slot
      const int i = g.esrc[y], j = g.edst[y], pj = jb.device_of[j];
      if (jb.device_of[i] != pj) jb.cache[static_cast<int64_t>(i) * n + pj] = INT64_MAX;
    }
    __syncwarp();
    for (int y = lane; y < g.E; y += 32) {
      const int i = g.esrc[y], j = g.edst[y], pj = jb.device_of[j];
      if (jb.device_of[i] != pj)
        atomicMin(reinterpret_cast<long long *>(jb.cache + static_cast<int64_t>(i) * n + pj),
                  (static_cast<long long>(tpos[j]) << 32) | g.inpos[y]);
    }
    __syncwarp();
    for (int d = 0; d < n; ++d) {
      const int o = jb.exec_off[d], len = jb.exec_off[d + 1] - o;
      int64_t prev = 0;
      for (int b = 0; b < len; b += 32) {
        const int idx = b + lane;
        int64_t A = 0, kk = 0;
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
        int64_t al = kk, be = A + kk;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
          const int64_t a2 = __shfl_up_sync(kFull, al, off), b2 = __shfl_up_sync(kFull, be, off);
          if (lane >= off) {
            be = max64(b2 + al, be);
            al = a2 + al;
          }
        }
        const int64_t f = max64(prev + al, be);
        if (idx < len) {
          jb.start[j] = f - kk;
          jb.finish[j] = f;
        }
        prev = __shfl_sync(kFull, f, 31);
        __syncwarp();
      }
    }
    if (lane == 0) {
      jb.stats[0] = jb.stats[1] = jb.stats[2] = 0;
      set_err(jb.err, kOk, E_NONE, 0, 0);
    }
    return;
  }
  if (lane == 0) {
    // schedule estimate (placers.cpp:350-362), sequential comm: the queue
    // tails make it a fold in topo order; every device_of is set before it
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
void launch_small(const DJob *jobs, const int32_t *order, int n_etf, int n_gen, const DGraph *graphs,
                  const DPrep *preps, int maxn, bool prof, cudaStream_t s, cudaStream_t s_gen);
void launch_big_seq(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                    int maxn, bool prof, cudaStream_t s);
void launch_rounds(const DJob *jobs, const int32_t *order, int njobs, const DGraph *graphs, const DPrep *preps,
                   int maxn, int list_len, cudaStream_t s);

void launch_prep_all(const DGraph *graphs_dev, const DPrep *preps_dev, int nprep, int max_ev, cudaStream_t s) {
  if (nprep <= 0 || max_ev <= 0) return;
  int x = (max_ev + 255) / 256;
  const int cap = nprep >= 1184 ? 1 : 1184 / nprep;
  if (x > cap) x = cap;
  for (int b = 0; b < nprep; b += 65535) {
    const int ny = nprep - b < 65535 ? nprep - b : 65535;
    k_prep_all<<<dim3(x, ny), 256, 0, s>>>(graphs_dev, preps_dev + b);
  }
}

void launch_fill(const FillChunk *table, int n, cudaStream_t s) {
  if (n > 0) k_fill<<<n < 148 * 8 ? n : 148 * 8, 256, 0, s>>>(table, n);
}

void launch_kahn(DGraph *graphs_dev, int32_t *const *queues_dev, int ngraphs, cudaStream_t s) {
  k_kahn<<<ngraphs, 512, 0, s>>>(graphs_dev, queues_dev);
}

// need_order: node indices by ascending (need, index), every graph of the
// plan in one segmented sort over the concatenated need arrays (stable, so
// equal needs keep ascending index order).
cudaError_t sort_needs_all(void *tmp, size_t &tmp_bytes, const int64_t *need, int64_t *keys_out, const int32_t *iota,
                           int32_t *order_out, int total, int nseg, const int32_t *seg_off, cudaStream_t s) {
  return cub::DeviceSegmentedSort::StableSortPairs(tmp, tmp_bytes, need, keys_out, iota, order_out, total, nseg,
                                                   seg_off, seg_off + 1, s);
}

void launch_placers(const DJob *jobs, const int32_t *order, int n_small, int n_etf, int n_bpar, int n_bseq,
                    int njobs, const DGraph *graphs, const DPrep *preps, int maxn, bool any_topo, bool prof,
                    int list_len, cudaStream_t s_small, cudaStream_t s_big) {
  // big problems (CTA-wide kernels) on s_big, beside the small ones (one
  // warp per job, four per CTA) on s_small; every list is longest-first
  if (n_bpar) launch_rounds(jobs, order + n_small, n_bpar, graphs, preps, maxn, list_len, s_big);
  if (n_bseq) launch_big_seq(jobs, order + n_small + n_bpar, n_bseq, graphs, preps, maxn, prof, s_big);
  if (n_small) launch_small(jobs, order, n_etf, n_small - n_etf, graphs, preps, maxn, prof, s_small, s_big);
  if (any_topo) {
    constexpr int W = 4;
    k_place_topo<W><<<(njobs + W - 1) / W, 32 * W, static_cast<size_t>(W) * maxn * 56, s_small>>>(
        jobs, njobs, graphs, preps, maxn);
  }
}

}  // namespace bx

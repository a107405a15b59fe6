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

// Per producer: -1 when every out-edge carries the same byte count (so the
// same comm time: a cache arrival changes no consumer's parallel-mode key),
// else 0. k_prep_small, which runs after this for small-frontier jobs,
// refines it from the comm times and numbers the rest.
__device__ __forceinline__ void prep_uniform(const DGraph &g, const DPrep &pr, int tid, int nthreads) {
  for (int i = tid; i < g.V; i += nthreads) {
    const int b = g.out_off[i], e = g.out_off[i + 1];
    bool uni = true;
    for (int y = b + 1; y < e && uni; ++y) uni = g.ebytes[y] == g.ebytes[b];
    pr.nu[i] = uni ? -1 : 0;
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
  prep_uniform(g, pr, tid, nth);
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


// need_order: node indices by ascending (need, index), every graph of the
// plan in one segmented sort over the concatenated need arrays (stable, so
// equal needs keep ascending index order).
cudaError_t sort_needs_all(void *tmp, size_t &tmp_bytes, const int64_t *need, int64_t *keys_out, const int32_t *iota,
                           int32_t *order_out, int total, int nseg, const int32_t *seg_off, cudaStream_t s) {
  return cub::DeviceSegmentedSort::StableSortPairs(tmp, tmp_bytes, need, keys_out, iota, order_out, total, nseg,
                                                   seg_off, seg_off + 1, s);
}

void launch_placers(const DJob *jobs, const int32_t *order, int n_small, int n_etf, int n_bpar, int n_bseq,
                    int njobs, const DGraph *graphs, const DPrep *preps, int maxn, bool prof,
                    int list_len, cudaStream_t s_small, cudaStream_t s_big) {
  // big problems (CTA-wide kernels) on s_big, beside the small ones (one
  // warp per job, four per CTA) on s_small; every list is longest-first
  if (n_bpar) launch_rounds(jobs, order + n_small, n_bpar, graphs, preps, maxn, list_len, s_big);
  if (n_bseq) launch_big_seq(jobs, order + n_small + n_bpar, n_bseq, graphs, preps, maxn, prof, s_big);
  if (n_small) launch_small(jobs, order, n_etf, n_small - n_etf, graphs, preps, maxn, prof, s_small, s_big);
}

}  // namespace bx

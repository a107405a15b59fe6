// Reference functions the placer API exposes beside the entry points:
//
//   schedulable_time (placers.hpp:66-67, placers.cpp:43-91) — the earliest
//     start of node j on device p for a given partial schedule. Here it is
//     evaluated for a whole batch of (j, p) queries at once (the ready set x
//     device set of one scheduling step is the natural query), one thread
//     per query, reading the in-CSR and the state arrays with coalesced
//     loads.
//   critical_path_us (simulator.cpp:296-309) — the compute-weighted longest
//     path, as a level-synchronous peel (one CTA per graph, the same peel
//     k_kahn uses for meta_topo_order's CycleError).
//
// Sequential comm mode without a scratch copy of the queue tails: the
// estimate folds parents in ascending in-edge order, and each fresh
// transfer sets tail(q) = tail(p) = term with term >= both old tails. So
// tail(p) is a running maximum, and a queue q touched earlier holds a term
// that is <= the current tail(p) and >= its original value; hence
// max(tail(q), tail(p)) == max(tail0[q], tail(p)) at every step and one
// register carries the whole scratch state.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/baechi_b200.h"
#include "arena.hpp"
#include "bx_device.cuh"

namespace bx {
namespace {

struct StQuery {
  int count, V, n, mode;
  double ic, pb;
  const int32_t *in_off, *in_edge, *esrc;
  const int64_t *ebytes;
  const int32_t *device_of;
  const int64_t *finish, *cache, *dev_free, *tail;
  const int32_t *qj, *qp;
  int64_t *out;
  int32_t *bad;  // [0] first failing query + 1 (unplaced parent in sequential mode), [1] negative bytes
};

__global__ void k_schedulable_time(StQuery q) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= q.count) return;
  const int j = q.qj[i], p = q.qp[i];
  const int n = q.n;
  int64_t t = q.dev_free[p];
  int64_t tp = q.tail[p];  // running scratch tail(p) (sequential mode)
  for (int x = q.in_off[j]; x < q.in_off[j + 1]; ++x) {
    const int e = q.in_edge[x];
    const int src = q.esrc[e];
    const int dq = q.device_of[src];
    const int64_t fin = q.finish[src];
    int64_t term;
    if (dq == p) {
      term = fin;
    } else {
      const int64_t cached = q.cache[static_cast<int64_t>(src) * n + p];
      if (cached >= 0) {
        term = fin > cached ? fin : cached;
      } else {
        const int64_t b = q.ebytes[e];
        if (b < 0) {
          atomicMin(&q.bad[1], i);
          return;
        }
        const int64_t c = comm_time_exact(q.ic, q.pb, b);
        if (q.mode == 1) {
          term = fin + c;
        } else {
          if (dq < 0 || dq >= n) {  // the reference indexes tail(-1): undefined
            atomicMin(&q.bad[0], i);
            return;
          }
          int64_t begin = fin > q.tail[dq] ? fin : q.tail[dq];
          begin = begin > tp ? begin : tp;
          term = begin + c;
          tp = term;
        }
      }
    }
    t = t > term ? t : term;
  }
  q.out[i] = t;
}

struct CpArgs {
  int V;
  const int32_t *in_off, *in_edge, *esrc, *out_off, *edst;
  const int64_t *k;
  int32_t *indeg, *queue;  // [V], [2V]
  int64_t *ready;          // [V] max finish over processed parents
  unsigned long long *best;
  int32_t *peeled;
};

// One CTA: level L pops its frontier, finishes every node in it (all parents
// sit in earlier levels), raises its children's ready time and appends the
// children whose last parent it was. Rotating counters, one barrier a level.
__global__ void __launch_bounds__(1024) k_critical_path(CpArgs a) {
  __shared__ int s_n[3];
  __shared__ int s_total;
  __shared__ unsigned long long s_best;
  const int V = a.V;
  if (threadIdx.x == 0) {
    s_n[0] = s_n[1] = s_n[2] = 0;
    s_total = 0;
    s_best = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < V; j += blockDim.x) {
    const int d = a.in_off[j + 1] - a.in_off[j];
    a.indeg[j] = d;
    a.ready[j] = 0;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < V; j += blockDim.x)
    if (a.indeg[j] == 0) a.queue[atomicAdd(&s_n[0], 1)] = j;
  __syncthreads();
  unsigned long long best = 0;
  for (int L = 0;; ++L) {
    const int cnt = s_n[L % 3];
    if (cnt == 0) break;
    const int32_t *in = a.queue + ((L & 1) ? V : 0);
    int32_t *out = a.queue + ((L & 1) ? 0 : V);
    int *next = &s_n[(L + 1) % 3];
    if (threadIdx.x == 0) {
      s_total += cnt;
      s_n[(L + 2) % 3] = 0;
    }
    for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
      const int u = in[x];
      const int64_t done = a.ready[u] + a.k[u];
      best = max(best, static_cast<unsigned long long>(done < 0 ? 0 : done));
      for (int y = a.out_off[u]; y < a.out_off[u + 1]; ++y) {
        const int v = a.edst[y];
        atomicMax(reinterpret_cast<long long *>(&a.ready[v]), static_cast<long long>(done));
      }
    }
    __syncthreads();  // every ready[] raise of this level lands before the decrements publish children
    for (int x = threadIdx.x; x < cnt; x += blockDim.x) {
      const int u = in[x];
      for (int y = a.out_off[u]; y < a.out_off[u + 1]; ++y) {
        const int v = a.edst[y];
        if (atomicSub(&a.indeg[v], 1) == 1) out[atomicAdd(next, 1)] = v;
      }
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long v = __shfl_xor_sync(0xffffffffu, best, o);
    best = v > best ? v : best;
  }
  if ((threadIdx.x & 31) == 0) atomicMax(&s_best, best);
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.best = s_best;
    *a.peeled = s_total;
  }
}

void put(char *msg, int msglen, const std::string &s) {
  if (msg && msglen > 0) std::snprintf(msg, static_cast<size_t>(msglen), "%s", s.c_str());
}

}  // namespace
}  // namespace bx

using namespace bx;

#define AX_CUDA(call)                                                                              \
  do {                                                                                             \
    cudaError_t e_ = (call);                                                                       \
    if (e_ != cudaSuccess) {                                                                       \
      put(msg, msglen, std::string("CUDA error: ") + cudaGetErrorString(e_) + " at " #call);       \
      return BX_RUNTIME;                                                                           \
    }                                                                                              \
  } while (0)

extern "C" {

int bx_schedulable_time(const bx_graph *g, const bx_comm *cm, const bx_placer_state *st, int32_t count,
                        const int32_t *node, const int32_t *device, int64_t *out, char *msg, int msglen) {
  put(msg, msglen, "");
  if (count < 0 || st->n <= 0 || st->V != g->V) {
    put(msg, msglen, "placer state does not match the graph");
    return BX_VALIDATION;
  }
  for (int i = 0; i < count; ++i) {
    if (node[i] < 0 || node[i] >= g->V || device[i] < 0 || device[i] >= st->n) {
      put(msg, msglen, "schedulable_time: node or device out of range");
      return BX_VALIDATION;
    }
  }
  if (count == 0) return BX_OK;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    put(msg, msglen, "no CUDA device: the placement engine has no CPU fallback");
    return BX_RUNTIME;
  }
  const int64_t V = g->V, E = g->E, n = st->n;
  Arena &A = thread_arena();
  Layout L;
  const size_t o_in_off = L.take<int32_t>(V + 1), o_in_edge = L.take<int32_t>(E), o_esrc = L.take<int32_t>(E);
  const size_t o_eb = L.take<int64_t>(E), o_dev = L.take<int32_t>(V), o_fin = L.take<int64_t>(V);
  const size_t o_cache = L.take<int64_t>(V * n), o_free = L.take<int64_t>(n), o_tail = L.take<int64_t>(n);
  const size_t o_qj = L.take<int32_t>(count), o_qp = L.take<int32_t>(count), o_out = L.take<int64_t>(count);
  const size_t o_bad = L.take<int32_t>(2);
  char *base = nullptr;
  AX_CUDA(A.device(L.off, &base));
  std::vector<HostCopy> cp = {
      {base + o_in_off, g->in_off, 4 * size_t(V + 1)}, {base + o_in_edge, g->in_edge, 4 * size_t(E)},
      {base + o_esrc, g->esrc, 4 * size_t(E)},          {base + o_eb, g->tensor_bytes, 8 * size_t(E)},
      {base + o_dev, st->device_of, 4 * size_t(V)},     {base + o_fin, st->finish_us, 8 * size_t(V)},
      {base + o_cache, st->cache_arrival, 8 * size_t(V * n)}, {base + o_free, st->dev_free, 8 * size_t(n)},
      {base + o_tail, st->xfer_tail, 8 * size_t(n)},    {base + o_qj, node, 4 * size_t(count)},
      {base + o_qp, device, 4 * size_t(count)}};
  cudaStream_t s = A.stream();
  for (const HostCopy &c : cp)
    if (c.bytes) AX_CUDA(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, s));
  const int32_t init[2] = {INT32_MAX, INT32_MAX};
  AX_CUDA(cudaMemcpyAsync(base + o_bad, init, 8, cudaMemcpyHostToDevice, s));
  StQuery q;
  q.count = count;
  q.V = g->V;
  q.n = st->n;
  q.mode = st->mode;
  q.ic = cm->intercept_us;
  q.pb = cm->us_per_byte;
  q.in_off = reinterpret_cast<const int32_t *>(base + o_in_off);
  q.in_edge = reinterpret_cast<const int32_t *>(base + o_in_edge);
  q.esrc = reinterpret_cast<const int32_t *>(base + o_esrc);
  q.ebytes = reinterpret_cast<const int64_t *>(base + o_eb);
  q.device_of = reinterpret_cast<const int32_t *>(base + o_dev);
  q.finish = reinterpret_cast<const int64_t *>(base + o_fin);
  q.cache = reinterpret_cast<const int64_t *>(base + o_cache);
  q.dev_free = reinterpret_cast<const int64_t *>(base + o_free);
  q.tail = reinterpret_cast<const int64_t *>(base + o_tail);
  q.qj = reinterpret_cast<const int32_t *>(base + o_qj);
  q.qp = reinterpret_cast<const int32_t *>(base + o_qp);
  q.out = reinterpret_cast<int64_t *>(base + o_out);
  q.bad = reinterpret_cast<int32_t *>(base + o_bad);
  k_schedulable_time<<<(count + 255) / 256, 256, 0, s>>>(q);
  AX_CUDA(cudaGetLastError());
  int32_t bad[2];
  AX_CUDA(cudaMemcpyAsync(out, q.out, 8 * size_t(count), cudaMemcpyDeviceToHost, s));
  AX_CUDA(cudaMemcpyAsync(bad, q.bad, 8, cudaMemcpyDeviceToHost, s));
  AX_CUDA(cudaStreamSynchronize(s));
  if (bad[1] != INT32_MAX) {
    put(msg, msglen, "comm_time: negative byte count");  // cost_model.cpp:31-33
    return BX_VALIDATION;
  }
  if (bad[0] != INT32_MAX) {
    put(msg, msglen, "schedulable_time: a remote parent of node " + std::to_string(node[bad[0]]) +
                         " is unplaced (sequential mode needs its queue)");
    return BX_VALIDATION;
  }
  return BX_OK;
}

int bx_critical_path_us(const bx_graph *g, int64_t *out_us, char *msg, int msglen) {
  put(msg, msglen, "");
  *out_us = 0;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    put(msg, msglen, "no CUDA device: the placement engine has no CPU fallback");
    return BX_RUNTIME;
  }
  const int64_t V = g->V, E = g->E;
  if (V == 0) return BX_OK;
  Arena &A = thread_arena();
  Layout L;
  const size_t o_in_off = L.take<int32_t>(V + 1), o_in_edge = L.take<int32_t>(E), o_esrc = L.take<int32_t>(E);
  const size_t o_out_off = L.take<int32_t>(V + 1), o_edst = L.take<int32_t>(E), o_k = L.take<int64_t>(V);
  const size_t o_indeg = L.take<int32_t>(V), o_q = L.take<int32_t>(2 * V), o_ready = L.take<int64_t>(V);
  const size_t o_best = L.take<unsigned long long>(1), o_peeled = L.take<int32_t>(1);
  char *base = nullptr;
  AX_CUDA(A.device(L.off, &base));
  cudaStream_t s = A.stream();
  const HostCopy cp[] = {{base + o_in_off, g->in_off, 4 * size_t(V + 1)},
                         {base + o_in_edge, g->in_edge, 4 * size_t(E)},
                         {base + o_esrc, g->esrc, 4 * size_t(E)},
                         {base + o_out_off, g->out_off, 4 * size_t(V + 1)},
                         {base + o_edst, g->edst, 4 * size_t(E)},
                         {base + o_k, g->compute_us, 8 * size_t(V)}};
  for (const HostCopy &c : cp)
    if (c.bytes) AX_CUDA(cudaMemcpyAsync(c.dst, c.src, c.bytes, cudaMemcpyHostToDevice, s));
  CpArgs a;
  a.V = g->V;
  a.in_off = reinterpret_cast<const int32_t *>(base + o_in_off);
  a.in_edge = reinterpret_cast<const int32_t *>(base + o_in_edge);
  a.esrc = reinterpret_cast<const int32_t *>(base + o_esrc);
  a.out_off = reinterpret_cast<const int32_t *>(base + o_out_off);
  a.edst = reinterpret_cast<const int32_t *>(base + o_edst);
  a.k = reinterpret_cast<const int64_t *>(base + o_k);
  a.indeg = reinterpret_cast<int32_t *>(base + o_indeg);
  a.queue = reinterpret_cast<int32_t *>(base + o_q);
  a.ready = reinterpret_cast<int64_t *>(base + o_ready);
  a.best = reinterpret_cast<unsigned long long *>(base + o_best);
  a.peeled = reinterpret_cast<int32_t *>(base + o_peeled);
  k_critical_path<<<1, 1024, 0, s>>>(a);
  AX_CUDA(cudaGetLastError());
  unsigned long long best = 0;
  int32_t peeled = 0;
  AX_CUDA(cudaMemcpyAsync(&best, a.best, 8, cudaMemcpyDeviceToHost, s));
  AX_CUDA(cudaMemcpyAsync(&peeled, a.peeled, 4, cudaMemcpyDeviceToHost, s));
  AX_CUDA(cudaStreamSynchronize(s));
  if (peeled != g->V) {
    // meta_topo_order's CycleError (transforms.cpp:466-477): the nodes the
    // peel could not remove, by their groups' first base ids
    std::vector<int32_t> left(static_cast<size_t>(V));
    AX_CUDA(cudaMemcpy(left.data(), a.indeg, 4 * size_t(V), cudaMemcpyDeviceToHost));
    std::string m = "meta graph is cyclic; groups of base node ids {";
    bool first = true;
    for (int64_t i = 0; i < V; ++i) {
      if (left[i] <= 0) continue;
      const long long id = g->first_id ? static_cast<long long>(g->first_id[i]) : static_cast<long long>(i);
      m += (first ? "" : ", ") + std::to_string(id);
      first = false;
    }
    put(msg, msglen, m + "} remain");
    return BX_VALIDATION;
  }
  *out_us = static_cast<int64_t>(best);
  return BX_OK;
}

}  // extern "C"

// m-SCT's favourite-child LP: build_lp (proj/src/lp.cpp:14-79) and
// solve_relaxed (:124-278) restated in C++17/CUDA. K5: the whole
// interior-point loop (Mehrotra predictor-corrector on G z <= h, same scaling
// f = 100/max coef, same strictly feasible start, eta, tolerances and
// 200-iteration cap) runs on the device in ONE persistent CTA: G z and G^T v
// as CSR passes, the normal matrix N = G^T W G + reg I assembled into the
// value array of its Cholesky factor (per-entry contribution lists, a fixed
// summation order), a hand-written sparse Cholesky and the triangular solves
// for the predictor and the corrector — the role of the reference's Eigen
// SimplicialLDLT. The host only builds the LP once: rows in the reference's
// order, a minimum-degree ordering of N's graph (the w column, which couples
// every completion row, has the largest degree and is eliminated last, so it
// causes no fill), and the symbolic factor (column structures = the
// elimination graph's neighbourhoods), plus a per-column map of the
// right-looking updates (target position, source pair) when it fits a
// budget; beyond it the update of a column walks each target column's row
// list (a merge, no search). Eigen3 is absent from the image, so parity with
// the reference is at the reference tests' tolerance (test_lp.cpp), not bit
// level.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/baechi_b200.h"
#include "bx_device.cuh"

namespace {

struct Row {
  std::vector<std::pair<int, double>> e;  // (var, coef)
  double rhs;
};

struct Lp {
  int V = 0, E = 0;
  std::vector<double> k, c;
  std::vector<int> src, dst;
  std::vector<Row> rows;
  int completion = 0, precedence = 0, child = 0, parent = 0, bounds = 0;
  int nvars() const { return V + E + 1; }
  int s_var(int i) const { return i; }
  int x_var(int e) const { return V + e; }
  int w_var() const { return V + E; }
};

struct SolverFail : std::runtime_error {
  explicit SolverFail(const std::string &m) : std::runtime_error(m) {}
};

// build_lp (lp.cpp:14-79): rows in the reference's order.
Lp build_lp(const bx_graph &g, const bx_comm &cm) {
  Lp lp;
  lp.V = g.V;
  lp.E = g.E;
  for (int i = 0; i < g.V; ++i) lp.k.push_back(static_cast<double>(g.compute_us[i]));
  for (int e = 0; e < g.E; ++e) {
    lp.c.push_back(static_cast<double>(bx::comm_time_exact(cm.intercept_us, cm.us_per_byte, g.tensor_bytes[e])));
    lp.src.push_back(g.esrc[e]);
    lp.dst.push_back(g.edst[e]);
  }
  for (int i = 0; i < lp.V; ++i) {
    lp.rows.push_back({{{lp.s_var(i), 1.0}, {lp.w_var(), -1.0}}, -lp.k[i]});
    lp.completion++;
  }
  for (int e = 0; e < lp.E; ++e) {
    int i = lp.src[e], j = lp.dst[e];
    lp.rows.push_back({{{lp.s_var(i), 1.0}, {lp.s_var(j), -1.0}, {lp.x_var(e), lp.c[e]}}, -lp.k[i]});
    lp.precedence++;
  }
  for (int i = 0; i < lp.V; ++i) {
    int d = g.out_off[i + 1] - g.out_off[i];
    if (!d) continue;
    Row r;
    for (int e = g.out_off[i]; e < g.out_off[i + 1]; ++e) r.e.push_back({lp.x_var(e), -1.0});
    r.rhs = 1.0 - d;
    lp.rows.push_back(r);
    lp.child++;
  }
  for (int j = 0; j < lp.V; ++j) {
    int d = g.in_off[j + 1] - g.in_off[j];
    if (!d) continue;
    Row r;
    for (int x = g.in_off[j]; x < g.in_off[j + 1]; ++x) r.e.push_back({lp.x_var(g.in_edge[x]), -1.0});
    r.rhs = 1.0 - d;
    lp.rows.push_back(r);
    lp.parent++;
  }
  for (int i = 0; i < lp.V; ++i) lp.rows.push_back({{{lp.s_var(i), -1.0}}, 0.0});
  lp.rows.push_back({{{lp.w_var(), -1.0}}, 0.0});
  for (int e = 0; e < lp.E; ++e) lp.rows.push_back({{{lp.x_var(e), -1.0}}, 0.0});
  for (int e = 0; e < lp.E; ++e) lp.rows.push_back({{{lp.x_var(e), 1.0}}, 1.0});
  lp.bounds = lp.V + 1 + 2 * lp.E;
  return lp;
}

// tighten_starts (lp.cpp:87-120): longest path for a fixed x, padded.
void tighten_starts(const Lp &lp, const std::vector<double> &x, const std::vector<double> &k,
                    const std::vector<double> &c, double pad, std::vector<double> &s) {
  const int n = lp.V;
  std::vector<std::vector<int>> in(n), out(n);
  std::vector<int> indeg(n, 0);
  for (int e = 0; e < lp.E; ++e) {
    in[lp.dst[e]].push_back(e);
    out[lp.src[e]].push_back(e);
    indeg[lp.dst[e]]++;
  }
  std::vector<int> order, stack;
  for (int i = n - 1; i >= 0; --i)
    if (!indeg[i]) stack.push_back(i);
  while (!stack.empty()) {
    int u = stack.back();
    stack.pop_back();
    order.push_back(u);
    for (int e : out[u])
      if (--indeg[lp.dst[e]] == 0) stack.push_back(lp.dst[e]);
  }
  s.assign(n, pad);
  for (int u : order)
    for (int e : in[u]) s[u] = std::max(s[u], s[lp.src[e]] + k[lp.src[e]] + c[e] * x[e] + pad);
}

// ---- host: ordering and symbolic factor ----------------------------------------
// Minimum-degree elimination on N's graph (ties: smallest variable), with the
// elimination graph kept explicitly: eliminating v makes its neighbours a
// clique. The neighbourhood at elimination is exactly the row structure of
// L's column for v.
struct Symbolic {
  int m = 0;
  std::vector<int> perm, iperm;    // perm[k] = variable eliminated k-th
  std::vector<int> colptr, rowidx;  // L in CSC, permuted indices, diagonal first, rows ascending
};

// `last`: a vertex adjacent to nearly everything (the makespan variable w,
// in every completion row) is kept out of the elimination graph — merging
// its adjacency at every elimination would cost O(V) each — ordered last,
// and added to every column's structure (a superset: the extra entries stay
// zero in the factor).
Symbolic min_degree_symbolic(const std::vector<std::vector<int>> &adj0, int last) {
  Symbolic S;
  const int m = static_cast<int>(adj0.size());
  S.m = m;
  std::vector<std::vector<int>> adj(adj0), lst(m);
  if (last >= 0) {
    for (auto &l : adj) l.erase(std::remove(l.begin(), l.end(), last), l.end());
    adj[last].clear();
  }
  std::set<std::pair<int, int>> q;
  for (int v = 0; v < m; ++v)
    if (v != last) q.insert({static_cast<int>(adj[v].size()), v});
  std::vector<char> gone(m, 0);
  std::vector<int> merged;
  S.perm.reserve(m);
  while (!q.empty()) {
    if (q.begin()->first == static_cast<int>(q.size()) - 1) {
      // the remaining graph is a clique (every degree is the minimum): each
      // elimination would only drop one vertex, so order the rest as they
      // come (degree, index) and give each the vertices after it
      std::vector<int> rest;
      for (const auto &dv : q) rest.push_back(dv.second);
      for (size_t i = 0; i < rest.size(); ++i) {
        S.perm.push_back(rest[i]);
        lst[rest[i]].assign(rest.begin() + static_cast<long>(i) + 1, rest.end());
      }
      break;
    }
    const int v = q.begin()->second;
    q.erase(q.begin());
    gone[v] = 1;
    S.perm.push_back(v);
    std::vector<int> nb;
    nb.swap(adj[v]);
    lst[v] = nb;
    for (int u : nb) {
      // adj[u] := (adj[u] u nb) \ {u, v}
      q.erase({static_cast<int>(adj[u].size()), u});
      merged.clear();
      std::set_union(adj[u].begin(), adj[u].end(), nb.begin(), nb.end(), std::back_inserter(merged));
      adj[u].clear();
      for (int x : merged)
        if (x != u && x != v) adj[u].push_back(x);
      q.insert({static_cast<int>(adj[u].size()), u});
    }
  }
  if (last >= 0) S.perm.push_back(last);
  S.iperm.assign(m, 0);
  for (int k = 0; k < m; ++k) S.iperm[S.perm[k]] = k;
  S.colptr.assign(m + 1, 0);
  for (int k = 0; k < m; ++k) {
    const int v = S.perm[k];
    std::vector<int> rows;
    rows.reserve(lst[v].size());
    for (int u : lst[v]) rows.push_back(S.iperm[u]);
    if (last >= 0 && v != last) rows.push_back(m - 1);
    std::sort(rows.begin(), rows.end());
    S.rowidx.push_back(k);
    S.rowidx.insert(S.rowidx.end(), rows.begin(), rows.end());
    S.colptr[k + 1] = static_cast<int>(S.rowidx.size());
  }
  return S;
}

// position of row r in column c of L (binary search; the entry must exist)
int lpos(const Symbolic &S, int c, int r) {
  auto b = S.rowidx.begin() + S.colptr[c], e = S.rowidx.begin() + S.colptr[c + 1];
  auto it = std::lower_bound(b, e, r);
  if (it == e || *it != r) throw std::runtime_error("symbolic factor misses an entry");
  return static_cast<int>(it - S.rowidx.begin());
}

// ---- device: the IPM loop in one CTA ---------------------------------------------
constexpr int kLpThreads = 1024;
constexpr int kLpWarps = kLpThreads / 32;
constexpr int kSmallCol = 96;  // columns up to this many entries: warp 0 alone, no CTA barrier

struct LpDev {
  int nv, nr, wvar, m, nnzL, ntgt, max_it;
  double tol;
  const int *grp, *gcol;    // G, CSR by row
  const double *gval, *h;
  const int *tptr, *trow;   // G^T, CSR by variable
  const double *tval;
  const int *perm, *colptr, *rowidx;
  const int *tgt_pos, *tgt_ptr, *con_row;  // normal-matrix entries: position in L, contributions
  const double *con_coef;
  const int *is_diag;                        // [ntgt] 1 when the target is a diagonal entry
  // elimination-tree levels (leaves first): columns of one level are
  // independent in the factorization and in both triangular solves
  int nlev;
  const int *lev_ptr, *lev_col;
  const int *rs_ptr;                         // [m+1] row structure of L: row j's entries left of the diagonal
  const int2 *rs_ent;                        // (column k, position of L(j, k))
  // left-looking update lists per factor position (null when over budget:
  // then the sequential right-looking factorization with merge walks)
  const long long *upd_ptr;                  // [nnzL + 1]
  const int2 *upd;                           // L[t] -= L[x] * L[y]
  // dense tail: columns [tail_t, m) are full (the final clique of the
  // ordering), factored as a d x d dense block after the sparse columns:
  // Dm = A_tail minus the sparse columns' updates (their update lists), a
  // dense Cholesky, copied back into L
  int tail_t, tail_d;
  double *Dm;
  // entries (L positions) of each level's sparse columns whose update list
  // is short (one thread sums it) or long (one warp sums it); the tail's
  // long-list entries (L position, Dm index)
  const int *lev_sptr, *lev_sent, *lev_lptr, *lev_lent;
  int tail_nlong;
  const int *tail_long_p, *tail_long_x;
  double *z, *lam, *slack, *rd, *W, *rc, *tmp, *rhs, *dza, *dz, *dsa, *dla, *ds, *dl, *y, *L;
  int *status;     // 0 ok, 1 lost feasibility, 2 no convergence, 3 factorization failed
  int *iters;
  double *gap;
};

struct LpRed {
  double v[2][kLpWarps];
};

enum RedOp { R_SUM, R_MIN, R_MAX };

template <RedOp OP>
__device__ __forceinline__ double warp_red(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double y = __shfl_xor_sync(0xffffffffu, x, o);
    x = OP == R_SUM ? x + y : OP == R_MIN ? fmin(x, y) : fmax(x, y);
  }
  return x;
}

// block reduction, one barrier (alternating scratch rows)
template <RedOp OP>
__device__ __forceinline__ double block_red(LpRed &R, int &par, double x) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  x = warp_red<OP>(x);
  if (lane == 0) R.v[par][warp] = x;
  __syncthreads();
  double r = OP == R_SUM ? 0.0 : OP == R_MIN ? INFINITY : -INFINITY;
  for (int w = 0; w < kLpWarps; ++w) {  // fixed order: every thread gets the same bits
    const double t = R.v[par][w];
    r = OP == R_SUM ? r + t : OP == R_MIN ? fmin(r, t) : fmax(r, t);
  }
  par ^= 1;
  return r;
}

// out[r] = h[r] - (G v)[r]   (sign = -1, base = h)   or   out[r] = -(G v)[r]
__device__ void g_times(const LpDev &D, const double *v, const double *base, double *out) {
  for (int r = threadIdx.x; r < D.nr; r += kLpThreads) {
    double acc = 0.0;
    for (int q = D.grp[r]; q < D.grp[r + 1]; ++q) acc += D.gval[q] * v[D.gcol[q]];
    out[r] = base ? base[r] - acc : -acc;
  }
}

// out[v] = (G^T u)[v] + add(v)
__device__ void gt_times(const LpDev &D, const double *u, double *out, const double *sub, bool obj) {
  for (int v = threadIdx.x; v < D.nv; v += kLpThreads) {
    double acc = 0.0;
    for (int q = D.tptr[v]; q < D.tptr[v + 1]; ++q) acc += D.tval[q] * u[D.trow[q]];
    if (obj && v == D.wvar) acc += 1.0;
    out[v] = sub ? acc - sub[v] : acc;
  }
}

constexpr int kLongList = 16;  // update lists longer than this are summed by a warp

// sum of an entry's update products, lanes over the list, fixed-order tree
// reduction (every lane returns it)
__device__ __forceinline__ double list_sum(const LpDev &D, int p, int lane) {
  double acc = 0.0;
  for (long long q = D.upd_ptr[p] + lane; q < D.upd_ptr[p + 1]; q += 32) {
    const int2 xy = D.upd[q];
    acc += D.L[xy.x] * D.L[xy.y];
  }
  return warp_red<R_SUM>(acc);
}

// The dense tail (see LpDev): each entry starts from A minus its own list of
// sparse-column products (fixed order), then a right-looking dense Cholesky
// (one column per step, trailing update by warps over columns), copy back.
__device__ void dense_tail(const LpDev &D, int *s_fail) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = D.tail_t, d = D.tail_d;
  for (long long x = tid; x < static_cast<long long>(d) * d; x += kLpThreads) {
    const int i = static_cast<int>(x % d), j = static_cast<int>(x / d);
    if (i < j) continue;
    const int p = D.colptr[t + j] + (i - j);
    const long long q0 = D.upd_ptr[p], q1 = D.upd_ptr[p + 1];
    if (q1 - q0 > kLongList) continue;  // summed by a warp below
    double v = D.L[p];
    for (long long q = q0; q < q1; ++q) {
      const int2 xy = D.upd[q];
      v -= D.L[xy.x] * D.L[xy.y];
    }
    D.Dm[x] = v;
  }
  for (int e = warp; e < D.tail_nlong; e += kLpWarps) {
    const int p = D.tail_long_p[e];
    D.Dm[D.tail_long_x[e]] = D.L[p] - list_sum(D, p, lane);
  }
  __syncthreads();
  for (int j = 0; j < d; ++j) {
    double djj = D.Dm[static_cast<long long>(j) * d + j];
    if (!(djj > 0.0)) {
      if (tid == 0) *s_fail = 1;
      djj = 1.0;
    }
    const double sq = sqrt(djj), inv = 1.0 / sq;
    __syncthreads();  // every thread has read the pivot
    double *cj = D.Dm + static_cast<long long>(j) * d;
    for (int i = j + 1 + tid; i < d; i += kLpThreads) cj[i] *= inv;
    if (tid == 0) cj[j] = sq;
    __syncthreads();
    for (int c = j + 1 + warp; c < d; c += kLpWarps) {
      const double lc = cj[c];
      double *cc = D.Dm + static_cast<long long>(c) * d;
      for (int r = c + lane; r < d; r += 32) cc[r] -= cj[r] * lc;
    }
    __syncthreads();
  }
  for (long long x = tid; x < static_cast<long long>(d) * d; x += kLpThreads) {
    const int i = static_cast<int>(x % d), j = static_cast<int>(x / d);
    if (i >= j) D.L[D.colptr[t + j] + (i - j)] = D.Dm[x];
  }
  __syncthreads();
}

// N = G^T W G + reg I written into L's values (fill positions zeroed), then
// L L^T = N in place. With update lists: left-looking, one warp per column,
// the columns of an elimination-tree level in parallel (their subtrees are
// disjoint), one CTA barrier per level; each factor entry subtracts its own
// list of products in a fixed order (deterministic). Otherwise: right-looking
// column by column, each source column updating its target columns by merge
// walks (warp 0 alone for small columns). Returns false on a non-positive
// pivot.
__device__ bool factor(const LpDev &D, double reg, int *s_fail) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int p = tid; p < D.nnzL; p += kLpThreads) D.L[p] = 0.0;
  __syncthreads();
  for (int t = tid; t < D.ntgt; t += kLpThreads) {
    double acc = D.is_diag[t] ? reg : 0.0;
    for (int q = D.tgt_ptr[t]; q < D.tgt_ptr[t + 1]; ++q) acc += D.W[D.con_row[q]] * D.con_coef[q];
    D.L[D.tgt_pos[t]] = acc;
  }
  if (tid == 0) *s_fail = 0;
  __syncthreads();
  if (D.upd_ptr) {
    for (int lv = 0; lv < D.nlev; ++lv) {
      // every entry of the level's sparse columns minus its update products
      // (short lists: one thread each; long lists: one warp each) ...
      for (int i = D.lev_sptr[lv] + tid; i < D.lev_sptr[lv + 1]; i += kLpThreads) {
        const int p = D.lev_sent[i];
        double v = D.L[p];
        for (long long q = D.upd_ptr[p]; q < D.upd_ptr[p + 1]; ++q) {
          const int2 xy = D.upd[q];
          v -= D.L[xy.x] * D.L[xy.y];
        }
        D.L[p] = v;
      }
      for (int i = D.lev_lptr[lv] + warp; i < D.lev_lptr[lv + 1]; i += kLpWarps) {
        const int p = D.lev_lent[i];
        const double sum = list_sum(D, p, lane);
        if (lane == 0) D.L[p] -= sum;
      }
      __syncthreads();
      // ... then each column's pivot and scaling, one warp per column
      for (int c = D.lev_ptr[lv] + warp; c < D.lev_ptr[lv + 1]; c += kLpWarps) {
        const int k = D.lev_col[c];
        if (k >= D.tail_t) continue;  // the dense tail comes after every sparse column
        const int b = D.colptr[k], e = D.colptr[k + 1];
        double d = D.L[b];
        if (!(d > 0.0)) {
          if (lane == 0) *s_fail = 1;
          d = 1.0;
        }
        const double sd = sqrt(d), inv = 1.0 / sd;
        __syncwarp();
        for (int p = b + 1 + lane; p < e; p += 32) D.L[p] *= inv;
        if (lane == 0) D.L[b] = sd;
      }
      __syncthreads();
    }
    if (D.tail_d > 0) dense_tail(D, s_fail);
    return *s_fail == 0;
  }
  for (int k = 0; k < D.m; ++k) {
    const int b = D.colptr[k], e = D.colptr[k + 1];
    const bool small = e - b <= kSmallCol;
    if (small && warp != 0) continue;
    if (!small) __syncthreads();
    const int nth = small ? 32 : kLpThreads, me = small ? lane : tid;
    double d = D.L[b];
    if (!(d > 0.0)) {  // a non-positive pivot: flag it, keep the barrier pattern (it is uniform)
      if (me == 0) *s_fail = 1;
      d = 1.0;
    }
    const double sd = sqrt(d), inv = 1.0 / sd;
    for (int p = b + 1 + me; p < e; p += nth) D.L[p] *= inv;
    if (me == 0) D.L[b] = sd;
    if (small) __syncwarp();
    else __syncthreads();
    // target column a = rowidx[p1]; rows rowidx[p2] (p2 >= p1) sit in a's
    // sorted list: one merge walk per target column
    for (int p1 = b + 1 + me; p1 < e; p1 += nth) {
      const int a = D.rowidx[p1];
      const double l1 = D.L[p1];
      int q = D.colptr[a];
      for (int p2 = p1; p2 < e; ++p2) {
        const int r = D.rowidx[p2];
        while (D.rowidx[q] != r) ++q;
        D.L[q] -= l1 * D.L[p2];
      }
    }
    if (small) __syncwarp();
    else __syncthreads();
  }
  __syncthreads();
  return *s_fail == 0;
}

// out = N^{-1} rhs through L (perm space in D.y), level by level: forward
// solve leaves first (row j's entries are in its descendants' columns),
// backward solve roots first (column j's rows are its ancestors); one warp
// per column, dot products in a fixed order
__device__ void chol_solve(const LpDev &D, const double *rhs, double *out) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int k = tid; k < D.m; k += kLpThreads) D.y[k] = rhs[D.perm[k]];
  __syncthreads();
  for (int lv = 0; lv < D.nlev; ++lv) {
    for (int c = D.lev_ptr[lv] + warp; c < D.lev_ptr[lv + 1]; c += kLpWarps) {
      const int j = D.lev_col[c];
      double acc = 0.0;
      for (int q = D.rs_ptr[j] + lane; q < D.rs_ptr[j + 1]; q += 32) {
        const int2 kp = D.rs_ent[q];
        acc += D.L[kp.y] * D.y[kp.x];
      }
      acc = warp_red<R_SUM>(acc);
      if (lane == 0) D.y[j] = (D.y[j] - acc) / D.L[D.colptr[j]];
    }
    __syncthreads();
  }
  for (int lv = D.nlev - 1; lv >= 0; --lv) {
    for (int c = D.lev_ptr[lv] + warp; c < D.lev_ptr[lv + 1]; c += kLpWarps) {
      const int j = D.lev_col[c];
      const int b = D.colptr[j], e = D.colptr[j + 1];
      double acc = 0.0;
      for (int p = b + 1 + lane; p < e; p += 32) acc += D.L[p] * D.y[D.rowidx[p]];
      acc = warp_red<R_SUM>(acc);
      if (lane == 0) D.y[j] = (D.y[j] - acc) / D.L[b];
    }
    __syncthreads();
  }
  for (int k = tid; k < D.m; k += kLpThreads) out[D.perm[k]] = D.y[k];
  __syncthreads();
}

// largest step in [0, 1] keeping v + a dv >= 0 (min over dv < 0 of -v/dv)
__device__ double max_step(LpRed &R, int &par, const double *v, const double *dv, int n) {
  double a = 1.0;
  for (int i = threadIdx.x; i < n; i += kLpThreads)
    if (dv[i] < 0) a = fmin(a, -v[i] / dv[i]);
  return block_red<R_MIN>(R, par, a);
}

__global__ void __launch_bounds__(kLpThreads, 1) k_lp_ipm(LpDev D) {
  __shared__ LpRed R;
  __shared__ int s_fail;
  const int tid = threadIdx.x;
  int par = 0;
  const int nr = D.nr, nv = D.nv;
  int status = 0, iters = 0;
  double gap = 0.0;
  for (int it = 0; it < D.max_it; ++it) {
    g_times(D, D.z, D.h, D.slack);
    double mn = INFINITY;
    for (int r = tid; r < nr; r += kLpThreads) mn = fmin(mn, D.slack[r]);
    mn = block_red<R_MIN>(R, par, mn);
    if (mn <= 0) {
      status = 1;
      break;
    }
    gt_times(D, D.lam, D.rd, nullptr, true);
    double rdn = 0.0, sl = 0.0;
    for (int v = tid; v < nv; v += kLpThreads) rdn = fmax(rdn, fabs(D.rd[v]));
    for (int r = tid; r < nr; r += kLpThreads) sl += D.slack[r] * D.lam[r];
    rdn = block_red<R_MAX>(R, par, rdn);
    sl = block_red<R_SUM>(R, par, sl);
    const double mu = sl / nr;
    const double rel_gap = sl / (1.0 + fabs(D.z[D.wvar]));
    if (rel_gap <= D.tol && rdn <= sqrt(D.tol)) {
      iters = it;
      gap = rel_gap;
      break;
    }
    if (it == D.max_it - 1) {
      status = 2;
      break;
    }
    double wmax = 0.0;
    for (int r = tid; r < nr; r += kLpThreads) {
      const double w = D.lam[r] / D.slack[r];
      D.W[r] = w;
      wmax = fmax(wmax, w);
      D.rc[r] = D.lam[r] * D.slack[r];
      D.tmp[r] = D.rc[r] / D.slack[r];
    }
    wmax = block_red<R_MAX>(R, par, wmax);
    if (!factor(D, 1e-12 * fmax(1.0, wmax), &s_fail)) {
      status = 3;
      break;
    }
    // affine predictor
    gt_times(D, D.tmp, D.rhs, D.rd, false);
    __syncthreads();
    chol_solve(D, D.rhs, D.dza);
    g_times(D, D.dza, nullptr, D.dsa);
    __syncthreads();
    for (int r = tid; r < nr; r += kLpThreads) D.dla[r] = (-D.rc[r] - D.lam[r] * D.dsa[r]) / D.slack[r];
    __syncthreads();
    const double ap = max_step(R, par, D.slack, D.dsa, nr), ad = max_step(R, par, D.lam, D.dla, nr);
    double maff = 0.0;
    for (int r = tid; r < nr; r += kLpThreads) maff += (D.slack[r] + ap * D.dsa[r]) * (D.lam[r] + ad * D.dla[r]);
    maff = block_red<R_SUM>(R, par, maff) / nr;
    const double ratio = fmin(fmax(maff / mu, 0.0), 1.0);
    const double sigma = ratio * ratio * ratio;
    // corrector
    for (int r = tid; r < nr; r += kLpThreads) {
      D.rc[r] = D.lam[r] * D.slack[r] + D.dsa[r] * D.dla[r] - sigma * mu;
      D.tmp[r] = D.rc[r] / D.slack[r];
    }
    __syncthreads();
    gt_times(D, D.tmp, D.rhs, D.rd, false);
    __syncthreads();
    chol_solve(D, D.rhs, D.dz);
    g_times(D, D.dz, nullptr, D.ds);
    __syncthreads();
    for (int r = tid; r < nr; r += kLpThreads) D.dl[r] = (-D.rc[r] - D.lam[r] * D.ds[r]) / D.slack[r];
    __syncthreads();
    const double eta = mu > 1e-4 ? 0.95 : 0.999;
    const double alpha_p = fmin(1.0, eta * max_step(R, par, D.slack, D.ds, nr));
    const double alpha_d = fmin(1.0, eta * max_step(R, par, D.lam, D.dl, nr));
    for (int v = tid; v < nv; v += kLpThreads) D.z[v] += alpha_p * D.dz[v];
    for (int r = tid; r < nr; r += kLpThreads) D.lam[r] += alpha_d * D.dl[r];
    __syncthreads();
  }
  if (tid == 0) {
    *D.status = status;
    *D.iters = iters;
    *D.gap = gap;
  }
}

// device buffers of one solve (freed on every exit path)
struct DevBufs {
  std::vector<void *> p;
  ~DevBufs() {  // stream-ordered pool: repeated solves reuse the memory
    for (void *q : p) cudaFreeAsync(q, 0);
  }
  template <typename T>
  T *put(const std::vector<T> &v) {
    T *d = nullptr;
    const size_t bytes = sizeof(T) * std::max<size_t>(v.size(), 1);
    if (cudaMallocAsync(&d, bytes, 0) != cudaSuccess) throw std::runtime_error("cudaMalloc failed for the LP");
    p.push_back(d);
    if (!v.empty() && cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, 0) != cudaSuccess)
      throw std::runtime_error("cudaMemcpy failed for the LP");
    return d;
  }
  template <typename T>
  T *zeros(size_t n) {
    T *d = nullptr;
    if (cudaMallocAsync(&d, sizeof(T) * std::max<size_t>(n, 1), 0) != cudaSuccess)
      throw std::runtime_error("cudaMalloc failed for the LP");
    p.push_back(d);
    cudaMemsetAsync(d, 0, sizeof(T) * std::max<size_t>(n, 1), 0);
    return d;
  }
};

}  // namespace

extern "C" int bx_lp_solve(const bx_graph *graph, const bx_comm *cm, double tolerance, double *x_out,
                           double *s_out, bx_lp_info *info, char *msg, int msglen) {
  auto put = [&](const std::string &m) {
    if (msg && msglen > 0) std::snprintf(msg, static_cast<size_t>(msglen), "%s", m.c_str());
  };
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    put("no CUDA device: the B200 placement engine has no CPU fallback");
    return BX_RUNTIME;
  }
  try {
    for (int e = 0; e < graph->E; ++e)
      if (graph->tensor_bytes[e] < 0) {
        put("comm_time: negative byte count");
        return BX_VALIDATION;
      }
    {
      // keep freed LP buffers in the stream-ordered pool (repeated solves
      // then allocate without going back to the driver)
      int dev = 0;
      cudaGetDevice(&dev);
      cudaMemPool_t pool;
      if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
        uint64_t keep = UINT64_MAX;
        cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
      }
    }
    const auto t_host0 = std::chrono::steady_clock::now();
    const Lp lp = build_lp(*graph, *cm);
    const int nv = lp.nvars(), nr = static_cast<int>(lp.rows.size());
    // rescale time units (lp.cpp:128-136)
    double maxc = 1.0;
    for (double v : lp.k) maxc = std::max(maxc, v);
    for (double v : lp.c) maxc = std::max(maxc, v);
    const double f = 100.0 / maxc;
    std::vector<double> ks(lp.k), cs(lp.c);
    for (double &v : ks) v *= f;
    for (double &v : cs) v *= f;
    const int time_rows = lp.completion + lp.precedence;
    // G (CSR by row, the reference's row order), h, and G^T (CSR by variable)
    std::vector<int> grp(nr + 1, 0), gcol;
    std::vector<double> gval, h(nr);
    for (int r = 0; r < nr; ++r) {
      const double scale = r < time_rows ? f : 1.0;
      for (const auto &ent : lp.rows[r].e) {
        const bool is_x = ent.first >= lp.V && ent.first < lp.V + lp.E;
        gcol.push_back(ent.first);
        gval.push_back(is_x ? ent.second * scale : ent.second);
      }
      grp[r + 1] = static_cast<int>(gcol.size());
      h[r] = lp.rows[r].rhs * scale;
    }
    std::vector<int> tptr(nv + 1, 0), trow(gcol.size());
    std::vector<double> tval(gcol.size());
    for (int c : gcol) tptr[c + 1]++;
    for (int v = 0; v < nv; ++v) tptr[v + 1] += tptr[v];
    {
      std::vector<int> fillp(tptr.begin(), tptr.end() - 1);
      for (int r = 0; r < nr; ++r)
        for (int q = grp[r]; q < grp[r + 1]; ++q) {
          trow[fillp[gcol[q]]] = r;
          tval[fillp[gcol[q]]++] = gval[q];
        }
    }
    // strictly feasible start (lp.cpp:158-184)
    std::vector<int> outdeg(lp.V, 0), indeg(lp.V, 0);
    for (int e = 0; e < lp.E; ++e) {
      outdeg[lp.src[e]]++;
      indeg[lp.dst[e]]++;
    }
    std::vector<double> z(nv, 0.0);
    for (int e = 0; e < lp.E; ++e) {
      const int ds = outdeg[lp.src[e]], dd = indeg[lp.dst[e]];
      const double need = std::max((ds - 1.0) / ds, (dd - 1.0) / dd);
      z[lp.x_var(e)] = need + (1.0 - need) / 2.0;
    }
    {
      std::vector<double> ones(lp.E, 1.0), s0;
      tighten_starts(lp, ones, ks, cs, 1.0, s0);
      double wmax = 1.0;
      for (int i = 0; i < lp.V; ++i) {
        z[lp.s_var(i)] = s0[i];
        wmax = std::max(wmax, s0[i] + ks[i]);
      }
      z[lp.w_var()] = wmax + 1.0;
    }
    // N's graph, ordering and symbolic factor
    std::vector<std::vector<int>> adj(nv);
    for (int r = 0; r < nr; ++r)
      for (int a = grp[r]; a < grp[r + 1]; ++a)
        for (int b = grp[r]; b < grp[r + 1]; ++b)
          if (gcol[a] != gcol[b]) adj[gcol[a]].push_back(gcol[b]);
    for (auto &l : adj) {
      std::sort(l.begin(), l.end());
      l.erase(std::unique(l.begin(), l.end()), l.end());
    }
    const Symbolic S = min_degree_symbolic(adj, lp.w_var());
    adj.clear();
    adj.shrink_to_fit();
    // normal-matrix entries (lower triangle, permuted) -> L positions, each
    // with its (row, g_a g_b) contributions in row order
    struct Con {
      int pos, row;
      double coef;
    };
    std::vector<Con> con;
    for (int r = 0; r < nr; ++r)
      for (int a = grp[r]; a < grp[r + 1]; ++a)
        for (int b = a; b < grp[r + 1]; ++b) {
          const int pa = S.iperm[gcol[a]], pb = S.iperm[gcol[b]];
          con.push_back({lpos(S, std::min(pa, pb), std::max(pa, pb)), r, gval[a] * gval[b]});
        }
    std::stable_sort(con.begin(), con.end(), [](const Con &x, const Con &y) { return x.pos < y.pos; });
    std::vector<int> tgt_pos, tgt_ptr{0}, con_row, is_diag;
    std::vector<double> con_coef;
    std::vector<char> diag_seen(nv, 0);
    for (size_t i = 0; i < con.size(); ++i) {
      if (i == 0 || con[i].pos != con[i - 1].pos) {
        if (i) tgt_ptr.push_back(static_cast<int>(con_row.size()));
        tgt_pos.push_back(con[i].pos);
      }
      con_row.push_back(con[i].row);
      con_coef.push_back(con[i].coef);
    }
    if (!con.empty()) tgt_ptr.push_back(static_cast<int>(con_row.size()));
    {
      std::vector<char> isd(S.rowidx.size(), 0);
      for (int k = 0; k < nv; ++k) isd[S.colptr[k]] = 1;
      for (int p : tgt_pos) {
        is_diag.push_back(isd[p]);
        if (isd[p]) diag_seen[S.rowidx[p]] = 1;
      }
      for (int k = 0; k < nv; ++k)  // a diagonal with no contribution still gets reg
        if (!diag_seen[k]) {
          tgt_pos.push_back(S.colptr[k]);
          tgt_ptr.push_back(tgt_ptr.back());
          is_diag.push_back(1);
        }
    }
    // elimination-tree levels (leaves = 0) and the row structure of L
    std::vector<int> lev(nv, 0);
    int nlev = nv > 0 ? 1 : 0;
    for (int k = 0; k < nv; ++k)
      if (S.colptr[k + 1] - S.colptr[k] > 1) {
        const int par = S.rowidx[S.colptr[k] + 1];  // etree parent = first row below the diagonal
        lev[par] = std::max(lev[par], lev[k] + 1);
        nlev = std::max(nlev, lev[par] + 1);
      }
    std::vector<int> lev_ptr(nlev + 1, 0), lev_col(nv);
    for (int k = 0; k < nv; ++k) lev_ptr[lev[k] + 1]++;
    for (int l = 0; l < nlev; ++l) lev_ptr[l + 1] += lev_ptr[l];
    {
      std::vector<int> at(lev_ptr.begin(), lev_ptr.end() - 1);
      for (int k = 0; k < nv; ++k) lev_col[at[lev[k]]++] = k;
    }
    std::vector<int> rs_ptr(nv + 1, 0);
    std::vector<int2> rs_ent;
    for (int k = 0; k < nv; ++k)
      for (int p = S.colptr[k] + 1; p < S.colptr[k + 1]; ++p) rs_ptr[S.rowidx[p] + 1]++;
    for (int j = 0; j < nv; ++j) rs_ptr[j + 1] += rs_ptr[j];
    rs_ent.resize(rs_ptr[nv]);
    {
      std::vector<int> at(rs_ptr.begin(), rs_ptr.end() - 1);
      for (int k = 0; k < nv; ++k)  // k ascending: each row's entries in column order
        for (int p = S.colptr[k] + 1; p < S.colptr[k + 1]; ++p) rs_ent[at[S.rowidx[p]]++] = make_int2(k, p);
    }
    // dense tail: the longest run of full columns at the end (>= 64 of them)
    int tail_t = nv;
    while (tail_t > 0 && S.colptr[tail_t] - S.colptr[tail_t - 1] == nv - (tail_t - 1)) --tail_t;
    if (nv - tail_t < 64) tail_t = nv;
    const int tail_d = nv - tail_t;
    // left-looking update lists (per target entry of a sparse column, sources
    // in column order) when they fit the budget
    long long npairs = 0;
    for (int k = 0; k < tail_t; ++k) {
      const long long c = S.colptr[k + 1] - S.colptr[k] - 1;
      npairs += c * (c + 1) / 2;
    }
    constexpr long long kPairBudget = 96ll << 20;
    const size_t nnzL = S.rowidx.size();
    std::vector<long long> upd_ptr;
    std::vector<int2> upd;
    if (npairs <= kPairBudget) {
      upd_ptr.assign(nnzL + 1, 0);
      std::vector<int> tpos(static_cast<size_t>(npairs));
      size_t x = 0;
      for (int k = 0; k < tail_t; ++k) {
        const int b = S.colptr[k], e = S.colptr[k + 1];
        for (int p1 = b + 1; p1 < e; ++p1) {
          // rows rowidx[p2] (p2 >= p1) of target column rowidx[p1]: a merge walk
          int q = S.colptr[S.rowidx[p1]];
          for (int p2 = p1; p2 < e; ++p2) {
            while (S.rowidx[q] != S.rowidx[p2]) ++q;
            tpos[x++] = q;
            upd_ptr[q + 1]++;
          }
        }
      }
      for (size_t t = 0; t < nnzL; ++t) upd_ptr[t + 1] += upd_ptr[t];
      upd.resize(static_cast<size_t>(npairs));
      std::vector<long long> at(upd_ptr.begin(), upd_ptr.end() - 1);
      x = 0;
      for (int k = 0; k < tail_t; ++k) {
        const int b = S.colptr[k], e = S.colptr[k + 1];
        for (int p1 = b + 1; p1 < e; ++p1)
          for (int p2 = p1; p2 < e; ++p2) upd[at[tpos[x++]]++] = make_int2(p1, p2);
      }
    }
    // per level: the sparse columns' entries split by update-list length;
    // the tail's long-list entries
    std::vector<int> lev_sptr{0}, lev_sent, lev_lptr{0}, lev_lent, tail_long_p, tail_long_x;
    if (!upd_ptr.empty()) {
      constexpr long long kLong = 16;  // == kLongList
      for (int l = 0; l < nlev; ++l) {
        for (int c = lev_ptr[l]; c < lev_ptr[l + 1]; ++c) {
          const int k = lev_col[c];
          if (k >= tail_t) continue;
          for (int p = S.colptr[k]; p < S.colptr[k + 1]; ++p)
            (upd_ptr[p + 1] - upd_ptr[p] > kLong ? lev_lent : lev_sent).push_back(p);
        }
        lev_sptr.push_back(static_cast<int>(lev_sent.size()));
        lev_lptr.push_back(static_cast<int>(lev_lent.size()));
      }
      for (int j = 0; j < tail_d; ++j)
        for (int i = j; i < tail_d; ++i) {
          const int p = S.colptr[tail_t + j] + (i - j);
          if (upd_ptr[p + 1] - upd_ptr[p] > kLong) {
            tail_long_p.push_back(p);
            tail_long_x.push_back(j * tail_d + i);
          }
        }
    }
    // device side
    DevBufs B;
    LpDev D{};
    D.nv = nv;
    D.nr = nr;
    D.wvar = lp.w_var();
    D.m = nv;
    D.nnzL = static_cast<int>(S.rowidx.size());
    D.ntgt = static_cast<int>(tgt_pos.size());
    D.max_it = 200;
    D.tol = tolerance;
    D.grp = B.put(grp);
    D.gcol = B.put(gcol);
    D.gval = B.put(gval);
    D.h = B.put(h);
    D.tptr = B.put(tptr);
    D.trow = B.put(trow);
    D.tval = B.put(tval);
    D.perm = B.put(S.perm);
    D.colptr = B.put(S.colptr);
    D.rowidx = B.put(S.rowidx);
    D.tgt_pos = B.put(tgt_pos);
    D.tgt_ptr = B.put(tgt_ptr);
    D.con_row = B.put(con_row);
    D.con_coef = B.put(con_coef);
    D.is_diag = B.put(is_diag);
    D.nlev = nlev;
    D.lev_ptr = B.put(lev_ptr);
    D.lev_col = B.put(lev_col);
    D.rs_ptr = B.put(rs_ptr);
    D.rs_ent = B.put(rs_ent);
    D.upd_ptr = upd_ptr.empty() ? nullptr : B.put(upd_ptr);
    D.upd = upd_ptr.empty() ? nullptr : B.put(upd);
    // the sequential fallback factors every column itself (no dense tail)
    D.tail_t = upd_ptr.empty() ? nv : tail_t;
    D.tail_d = upd_ptr.empty() ? 0 : tail_d;
    D.Dm = B.zeros<double>(static_cast<size_t>(D.tail_d) * static_cast<size_t>(D.tail_d));
    D.lev_sptr = B.put(lev_sptr);
    D.lev_sent = B.put(lev_sent);
    D.lev_lptr = B.put(lev_lptr);
    D.lev_lent = B.put(lev_lent);
    D.tail_nlong = static_cast<int>(tail_long_p.size());
    D.tail_long_p = B.put(tail_long_p);
    D.tail_long_x = B.put(tail_long_x);
    D.z = B.put(z);
    D.lam = B.put(std::vector<double>(nr, 1.0));
    D.slack = B.zeros<double>(nr);
    D.rd = B.zeros<double>(nv);
    D.W = B.zeros<double>(nr);
    D.rc = B.zeros<double>(nr);
    D.tmp = B.zeros<double>(nr);
    D.rhs = B.zeros<double>(nv);
    D.dza = B.zeros<double>(nv);
    D.dz = B.zeros<double>(nv);
    D.dsa = B.zeros<double>(nr);
    D.dla = B.zeros<double>(nr);
    D.ds = B.zeros<double>(nr);
    D.dl = B.zeros<double>(nr);
    D.y = B.zeros<double>(nv);
    D.L = B.zeros<double>(S.rowidx.size());
    D.status = B.zeros<int>(1);
    D.iters = B.zeros<int>(1);
    D.gap = B.zeros<double>(1);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const double host_ms =
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_host0).count();
    cudaEventRecord(e0);
    k_lp_ipm<<<1, kLpThreads>>>(D);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float dev_ms = 0.f;
    cudaEventElapsedTime(&dev_ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    int st = 0, iters = 0;
    double gap = 0;
    if (cudaMemcpy(&st, D.status, 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&iters, D.iters, 4, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(&gap, D.gap, 8, cudaMemcpyDeviceToHost) != cudaSuccess ||
        cudaMemcpy(z.data(), D.z, 8 * size_t(nv), cudaMemcpyDeviceToHost) != cudaSuccess)
      throw std::runtime_error(std::string("LP kernel: ") + cudaGetErrorString(cudaGetLastError()));
    if (st == 1) throw SolverFail("interior point lost strict feasibility");
    if (st == 2) throw SolverFail("LP did not converge within 200 iterations; consider rescaling profile times");
    if (st == 3) throw SolverFail("normal-equation factorization failed");
    // unscale: clip x, re-tighten starts under the final x (lp.cpp:266-276)
    std::vector<double> x(lp.E), s;
    for (int e = 0; e < lp.E; ++e) x[e] = std::clamp(z[lp.x_var(e)], 0.0, 1.0);
    tighten_starts(lp, x, lp.k, lp.c, 0.0, s);
    double w = 0;
    for (int i = 0; i < lp.V; ++i) w = std::max(w, s[i] + lp.k[i]);
    for (int e = 0; e < lp.E; ++e) x_out[e] = x[e];
    if (s_out)
      for (int i = 0; i < lp.V; ++i) s_out[i] = s[i];
    if (info) {
      info->iterations = iters;
      info->rel_gap = gap;
      info->w = w;
      info->num_rows = nr;
      info->completion_rows = lp.completion;
      info->precedence_rows = lp.precedence;
      info->child_rows = lp.child;
      info->parent_rows = lp.parent;
      info->bound_rows = lp.bounds;
      info->host_ms = host_ms;
      info->device_ms = dev_ms;
      info->factor_nnz = static_cast<int64_t>(S.rowidx.size());
      info->update_pairs = upd_ptr.empty() ? 0 : npairs;
    }
    put("");
    return BX_OK;
  } catch (const SolverFail &e) {
    put(e.what());
    return BX_SOLVER;
  } catch (const std::exception &e) {
    put(std::string("LP failure: ") + e.what());
    return BX_RUNTIME;
  }
}

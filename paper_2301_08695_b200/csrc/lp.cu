// m-SCT's favourite-child LP: build_lp (proj/src/lp.cpp:14-79) and
// solve_relaxed (:124-278) restated in C++17. The interior-point iteration
// (Mehrotra predictor-corrector on G z <= h, same scaling f = 100/max coef,
// same strictly feasible start, eta, tolerances and 200-iteration cap) runs on
// the host; the normal equations (G^T W G + reg I) dz = r are factored on the
// GPU once per iteration and solved for both the predictor and the corrector:
// dense Cholesky (cuSOLVER potrf/potrs, FP64) up to kDenseMax variables —
// the w column couples every completion row, so the factor fills in anyway —
// and cuSOLVER's sparse Cholesky with fill-reducing reorder beyond, the
// analogues of the reference's Eigen SimplicialLDLT. Eigen3 is absent from
// the image, so parity with the reference is at the reference tests'
// tolerance (test_lp.cpp), not bit level.
#include <cuda_runtime.h>
#include <cusolverDn.h>
#include <cusolverSp.h>
#include <cusparse.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <numeric>
#include <stdexcept>
#include <string>
#include <unordered_map>
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

// Sparse symmetric normal matrix G^T W G with a fixed pattern; values are
// refilled every iteration from per-row pair lists.
struct Normal {
  int m = 0;
  std::vector<int> rowptr, colind;
  std::vector<double> val;
  std::vector<int> diag;                              // position of (i, i)
  std::vector<std::vector<std::pair<int, double>>> contrib;  // per G row: (pos, G_ra*G_rb)
};

Normal normal_pattern(const std::vector<Row> &G, int nvars) {
  Normal N;
  N.m = nvars;
  std::vector<std::vector<int>> cols(nvars);
  for (const Row &r : G)
    for (const auto &a : r.e)
      for (const auto &b : r.e) cols[a.first].push_back(b.first);
  for (int i = 0; i < nvars; ++i) cols[i].push_back(i);  // regularised diagonal
  N.rowptr.push_back(0);
  for (int i = 0; i < nvars; ++i) {
    auto &c = cols[i];
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    N.colind.insert(N.colind.end(), c.begin(), c.end());
    N.rowptr.push_back(static_cast<int>(N.colind.size()));
  }
  N.val.assign(N.colind.size(), 0.0);
  auto pos = [&](int a, int b) {
    auto it = std::lower_bound(N.colind.begin() + N.rowptr[a], N.colind.begin() + N.rowptr[a + 1], b);
    return static_cast<int>(it - N.colind.begin());
  };
  N.diag.resize(nvars);
  for (int i = 0; i < nvars; ++i) N.diag[i] = pos(i, i);
  N.contrib.resize(G.size());
  for (size_t r = 0; r < G.size(); ++r)
    for (const auto &a : G[r].e)
      for (const auto &b : G[r].e) N.contrib[r].push_back({pos(a.first, b.first), a.second * b.second});
  return N;
}

constexpr int kDenseMax = 24576;  // 4.8 GB of FP64 factor at the limit

__global__ void k_scatter_dense(int nnz, const int *rowidx, const int *colind, const double *val, double *A, int m) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < nnz; i += gridDim.x * blockDim.x)
    A[static_cast<size_t>(colind[i]) * m + rowidx[i]] = val[i];  // column-major; the pattern is symmetric
}

struct Chol {  // device side of the normal-equation solves
  cusolverSpHandle_t h = nullptr;
  cusolverDnHandle_t hd = nullptr;
  cusparseMatDescr_t d = nullptr;
  int *rowptr = nullptr, *colind = nullptr, *rowidx = nullptr, *dinfo = nullptr;
  double *val = nullptr, *b = nullptr, *x = nullptr, *A = nullptr, *work = nullptr;
  int m = 0, nnz = 0, reorder = 3, lwork = 0;
  bool dense = false;
  ~Chol() {
    if (h) cusolverSpDestroy(h);
    if (hd) cusolverDnDestroy(hd);
    if (d) cusparseDestroyMatDescr(d);
    cudaFree(rowptr);
    cudaFree(colind);
    cudaFree(rowidx);
    cudaFree(dinfo);
    cudaFree(val);
    cudaFree(b);
    cudaFree(x);
    cudaFree(A);
    cudaFree(work);
  }
  void init(const Normal &N) {
    m = N.m;
    nnz = static_cast<int>(N.colind.size());
    dense = m <= kDenseMax;
    if (cudaMalloc(&rowptr, 4 * size_t(m + 1)) || cudaMalloc(&colind, 4 * size_t(nnz)) ||
        cudaMalloc(&val, 8 * size_t(nnz)) || cudaMalloc(&b, 8 * size_t(m)) || cudaMalloc(&x, 8 * size_t(m)))
      throw std::runtime_error("cudaMalloc failed for the normal equations");
    cudaMemcpy(rowptr, N.rowptr.data(), 4 * size_t(m + 1), cudaMemcpyHostToDevice);
    cudaMemcpy(colind, N.colind.data(), 4 * size_t(nnz), cudaMemcpyHostToDevice);
    if (dense) {
      std::vector<int> ri(nnz);
      for (int r = 0; r < m; ++r)
        for (int q = N.rowptr[r]; q < N.rowptr[r + 1]; ++q) ri[q] = r;
      if (cusolverDnCreate(&hd) != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error("cusolverDnCreate failed");
      if (cudaMalloc(&rowidx, 4 * size_t(nnz)) || cudaMalloc(&A, 8 * size_t(m) * size_t(m)) ||
          cudaMalloc(&dinfo, sizeof(int)))
        throw std::runtime_error("cudaMalloc failed for the dense normal equations");
      cudaMemcpy(rowidx, ri.data(), 4 * size_t(nnz), cudaMemcpyHostToDevice);
      if (cusolverDnDpotrf_bufferSize(hd, CUBLAS_FILL_MODE_LOWER, m, A, m, &lwork) != CUSOLVER_STATUS_SUCCESS ||
          cudaMalloc(&work, 8 * size_t(std::max(lwork, 1))))
        throw std::runtime_error("potrf workspace");
    } else {
      if (cusolverSpCreate(&h) != CUSOLVER_STATUS_SUCCESS) throw std::runtime_error("cusolverSpCreate failed");
      cusparseCreateMatDescr(&d);
      cusparseSetMatType(d, CUSPARSE_MATRIX_TYPE_GENERAL);
      cusparseSetMatIndexBase(d, CUSPARSE_INDEX_BASE_ZERO);
    }
  }
  // new values for this iteration; the dense path factors here, once
  void load(const std::vector<double> &v) {
    cudaMemcpy(val, v.data(), 8 * size_t(nnz), cudaMemcpyHostToDevice);
    if (!dense) return;
    cudaMemset(A, 0, 8 * size_t(m) * size_t(m));
    const int blocks = std::min((nnz + 255) / 256, 4096);
    k_scatter_dense<<<std::max(blocks, 1), 256>>>(nnz, rowidx, colind, val, A, m);
    int info = 0;
    if (cusolverDnDpotrf(hd, CUBLAS_FILL_MODE_LOWER, m, A, m, work, lwork, dinfo) != CUSOLVER_STATUS_SUCCESS ||
        cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess || info != 0)
      throw SolverFail("normal-equation factorization failed");
  }
  void solve(const std::vector<double> &rhs, std::vector<double> &out) {
    cudaMemcpy(b, rhs.data(), 8 * size_t(m), cudaMemcpyHostToDevice);
    out.resize(m);
    if (dense) {
      int info = 0;
      if (cusolverDnDpotrs(hd, CUBLAS_FILL_MODE_LOWER, m, 1, A, m, b, m, dinfo) != CUSOLVER_STATUS_SUCCESS ||
          cudaMemcpy(&info, dinfo, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess || info != 0)
        throw SolverFail("normal-equation factorization failed");
      cudaMemcpy(out.data(), b, 8 * size_t(m), cudaMemcpyDeviceToHost);
      return;
    }
    int singular = -1;
    cusolverStatus_t st = cusolverSpDcsrlsvchol(h, m, nnz, d, val, rowptr, colind, b, 1e-14, reorder, x, &singular);
    if (st != CUSOLVER_STATUS_SUCCESS && reorder != 1) {  // older ordering codes only
      reorder = 1;
      st = cusolverSpDcsrlsvchol(h, m, nnz, d, val, rowptr, colind, b, 1e-14, reorder, x, &singular);
    }
    if (st != CUSOLVER_STATUS_SUCCESS || singular >= 0) throw SolverFail("normal-equation factorization failed");
    cudaMemcpy(out.data(), x, 8 * size_t(m), cudaMemcpyDeviceToHost);
  }
};

double dot(const std::vector<double> &a, const std::vector<double> &b) {
  double s = 0;
  for (size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

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
    std::vector<Row> G(lp.rows);
    std::vector<double> h(nr);
    for (int r = 0; r < nr; ++r) {
      double scale = r < time_rows ? f : 1.0;
      for (auto &ent : G[r].e) {
        bool is_x = ent.first >= lp.V && ent.first < lp.V + lp.E;
        if (is_x) ent.second *= scale;
      }
      h[r] = lp.rows[r].rhs * scale;
    }
    std::vector<double> cobj(nv, 0.0);
    cobj[lp.w_var()] = 1.0;
    // strictly feasible start (lp.cpp:158-184)
    std::vector<int> outdeg(lp.V, 0), indeg(lp.V, 0);
    for (int e = 0; e < lp.E; ++e) {
      outdeg[lp.src[e]]++;
      indeg[lp.dst[e]]++;
    }
    std::vector<double> z(nv, 0.0);
    for (int e = 0; e < lp.E; ++e) {
      int ds = outdeg[lp.src[e]], dd = indeg[lp.dst[e]];
      double need = std::max((ds - 1.0) / ds, (dd - 1.0) / dd);
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
    auto Gz = [&](const std::vector<double> &v) {
      std::vector<double> out(nr, 0.0);
      for (int r = 0; r < nr; ++r)
        for (const auto &ent : G[r].e) out[r] += ent.second * v[ent.first];
      return out;
    };
    auto Gtv = [&](const std::vector<double> &v) {
      std::vector<double> out(nv, 0.0);
      for (int r = 0; r < nr; ++r)
        for (const auto &ent : G[r].e) out[ent.first] += ent.second * v[r];
      return out;
    };
    Normal N = normal_pattern(G, nv);
    Chol chol;
    chol.init(N);
    std::vector<double> lambda(nr, 1.0), slack(nr);
    int iters = 0;
    double gap = 0;
    const int kMax = 200;
    for (int it = 0; it < kMax; ++it) {
      std::vector<double> gz = Gz(z);
      double mn = 1e300;
      for (int r = 0; r < nr; ++r) {
        slack[r] = h[r] - gz[r];
        mn = std::min(mn, slack[r]);
      }
      if (mn <= 0) throw SolverFail("interior point lost strict feasibility");
      std::vector<double> rd = Gtv(lambda);
      double rdn = 0;
      for (int i = 0; i < nv; ++i) {
        rd[i] += cobj[i];
        rdn = std::max(rdn, std::fabs(rd[i]));
      }
      const double sl = dot(slack, lambda);
      const double mu = sl / nr;
      const double rel_gap = sl / (1.0 + std::fabs(z[lp.w_var()]));
      if (rel_gap <= tolerance && rdn <= std::sqrt(tolerance)) {
        iters = it;
        gap = rel_gap;
        break;
      }
      if (it == kMax - 1)
        throw SolverFail("LP did not converge within 200 iterations; consider rescaling profile times");
      // normal matrix values
      std::vector<double> W(nr);
      double wmax = 0;
      for (int r = 0; r < nr; ++r) {
        W[r] = lambda[r] / slack[r];
        wmax = std::max(wmax, W[r]);
      }
      std::fill(N.val.begin(), N.val.end(), 0.0);
      for (int r = 0; r < nr; ++r)
        for (const auto &pc : N.contrib[r]) N.val[pc.first] += W[r] * pc.second;
      const double reg = 1e-12 * std::max(1.0, wmax);
      for (int i = 0; i < nv; ++i) N.val[N.diag[i]] += reg;
      chol.load(N.val);
      auto max_step = [](const std::vector<double> &v, const std::vector<double> &dv) {
        double a = 1.0;
        for (size_t i = 0; i < v.size(); ++i)
          if (dv[i] < 0) a = std::min(a, -v[i] / dv[i]);
        return a;
      };
      // affine predictor
      std::vector<double> rc(nr), tmp(nr);
      for (int r = 0; r < nr; ++r) {
        rc[r] = lambda[r] * slack[r];
        tmp[r] = rc[r] / slack[r];
      }
      std::vector<double> rhs = Gtv(tmp);
      for (int i = 0; i < nv; ++i) rhs[i] -= rd[i];
      std::vector<double> dz_aff;
      chol.solve(rhs, dz_aff);
      std::vector<double> ds_aff = Gz(dz_aff), dl_aff(nr);
      for (int r = 0; r < nr; ++r) {
        ds_aff[r] = -ds_aff[r];
        dl_aff[r] = (-rc[r] - lambda[r] * ds_aff[r]) / slack[r];
      }
      const double ap = max_step(slack, ds_aff), ad = max_step(lambda, dl_aff);
      double mu_aff = 0;
      for (int r = 0; r < nr; ++r) mu_aff += (slack[r] + ap * ds_aff[r]) * (lambda[r] + ad * dl_aff[r]);
      mu_aff /= nr;
      const double sigma = std::pow(std::clamp(mu_aff / mu, 0.0, 1.0), 3.0);
      // corrector
      for (int r = 0; r < nr; ++r) {
        rc[r] = lambda[r] * slack[r] + ds_aff[r] * dl_aff[r] - sigma * mu;
        tmp[r] = rc[r] / slack[r];
      }
      rhs = Gtv(tmp);
      for (int i = 0; i < nv; ++i) rhs[i] -= rd[i];
      std::vector<double> dz;
      chol.solve(rhs, dz);
      std::vector<double> ds = Gz(dz), dl(nr);
      for (int r = 0; r < nr; ++r) {
        ds[r] = -ds[r];
        dl[r] = (-rc[r] - lambda[r] * ds[r]) / slack[r];
      }
      const double eta = mu > 1e-4 ? 0.95 : 0.999;
      const double alpha_p = std::min(1.0, eta * max_step(slack, ds));
      const double alpha_d = std::min(1.0, eta * max_step(lambda, dl));
      for (int i = 0; i < nv; ++i) z[i] += alpha_p * dz[i];
      for (int r = 0; r < nr; ++r) lambda[r] += alpha_d * dl[r];
    }
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

// Weighted-quadrature Galerkin operator (eq:WQapprox P:195-199, eq:Q P:192):
//
//   (A_wq)_ij = sum_{alpha,beta} sum_q c_{alpha beta}(x_q) w^{alpha beta}_{iq} d_beta B^_j(x_q),
//   c = Q(xi) = det(J) J^{-1} J^{-T} (K = I),  w^{alpha beta}_{iq} = prod_l w_l^{(a_l b_l)}_{i_l q_l},
//   a_l = [l = alpha], b_l = [l = beta],
//
// stored in the tensor-window layout of the collocation operator (windows |i_l - j_l| <= p), so the same
// matvec kernel, FD preconditioner (symmetric 1D Galerkin pencils, eq:univariateWQ) and Krylov solvers
// serve it.  The 1D rule follows DESIGN.md reading 18 (the oracle's definition, implemented here
// independently): points = knot-span endpoints and midpoints (+ quarter points of the first / last p
// elements for rows whose moment system is inconsistent on the base set); per row and derivative pair
// (a, b) the minimum-norm weights on the points of supp(B_i) with
//   sum_q w^{ab}_{iq} B_j^{(b)}(x_q) = int B_i^{(a)} B_j^{(b)}  for every interior j with |i - j| <= p.
// Setup only (not on the timed path): the rule on the host, Q on the device point grid, then one thread
// per row contracts direction by direction (sum factorisation) into the row's (2p+1)^d window values.
#include <cmath>
#include <cstring>
#include <set>
#include <vector>

#include "bspline.h"
#include "common.cuh"
#include "geometry.cuh"

using namespace fdiga;

namespace {

// Gauss-Legendre nodes / weights on [-1, 1] (Newton on P_q)
void gauss_legendre(int q, std::vector<double>& x, std::vector<double>& w) {
  x.assign(q, 0.0);
  w.assign(q, 0.0);
  for (int i = 0; i < q; ++i) {
    double z = std::cos(M_PI * (i + 0.75) / (q + 0.5)), dp = 0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = 0.0;
      for (int k = 1; k <= q; ++k) {
        const double p2 = p1;
        p1 = p0;
        p0 = ((2.0 * k - 1.0) * z * p1 - (k - 1.0) * p2) / k;
      }
      dp = q * (z * p0 - p1) / (z * z - 1.0);
      const double dz = p0 / dp;
      z -= dz;
      if (std::fabs(dz) < 1e-16) break;
    }
    x[i] = z;
    w[i] = 2.0 / ((1.0 - z * z) * dp * dp);
  }
}

// Minimum-norm solution of the consistent system B w = m (B: nj x nq row-major) as w = B^T y,
// (B B^T) y = m by Gaussian elimination with complete pivoting; rank-deficient directions get y = 0.
bool min_norm(const std::vector<double>& B, int nj, int nq, const std::vector<double>& m, std::vector<double>& w) {
  std::vector<double> G((size_t)nj * nj, 0.0), r(m);
  for (int a = 0; a < nj; ++a)
    for (int b = 0; b < nj; ++b) {
      double s = 0;
      for (int q = 0; q < nq; ++q) s += B[a * nq + q] * B[b * nq + q];
      G[a * nj + b] = s;
    }
  double gmax = 0;
  for (int a = 0; a < nj; ++a) gmax = std::max(gmax, std::fabs(G[a * nj + a]));
  std::vector<int> col(nj);
  for (int a = 0; a < nj; ++a) col[a] = a;
  int rank = 0;
  for (int k = 0; k < nj; ++k) {
    int pr = k, pc = k;
    double best = 0;
    for (int a = k; a < nj; ++a)
      for (int b = k; b < nj; ++b)
        if (std::fabs(G[a * nj + b]) > best) {
          best = std::fabs(G[a * nj + b]);
          pr = a;
          pc = b;
        }
    if (best <= 1e-13 * gmax) break;
    for (int b = 0; b < nj; ++b) std::swap(G[k * nj + b], G[pr * nj + b]);
    std::swap(r[k], r[pr]);
    for (int a = 0; a < nj; ++a) std::swap(G[a * nj + k], G[a * nj + pc]);
    std::swap(col[k], col[pc]);
    for (int a = k + 1; a < nj; ++a) {
      const double f = G[a * nj + k] / G[k * nj + k];
      for (int b = k; b < nj; ++b) G[a * nj + b] -= f * G[k * nj + b];
      r[a] -= f * r[k];
    }
    ++rank;
  }
  std::vector<double> yp(nj, 0.0), y(nj, 0.0);
  for (int k = rank - 1; k >= 0; --k) {
    double s = r[k];
    for (int b = k + 1; b < rank; ++b) s -= G[k * nj + b] * yp[b];
    yp[k] = s / G[k * nj + k];
  }
  for (int k = 0; k < nj; ++k) y[col[k]] = yp[k];
  w.assign(nq, 0.0);
  for (int q = 0; q < nq; ++q)
    for (int a = 0; a < nj; ++a) w[q] += B[a * nq + q] * y[a];
  double res = 0, mn = 0;
  for (int a = 0; a < nj; ++a) {
    double s = -m[a];
    for (int q = 0; q < nq; ++q) s += B[a * nq + q] * w[q];
    res += s * s;
    mn += m[a] * m[a];
  }
  return std::sqrt(res) <= 1e-11 * std::max(1.0, std::sqrt(mn));
}

// The 1D rule: points, per-row point ranges, windows, and R^{ab}[i][jj][qq] = w^{ab}_{i,q} B^{(b)}_{j}(x_q)
struct WQRule {
  int64_t n = 0, nq = 0;
  int NJ = 0, QM = 0;  // window width bound 2p + 1, max points per row
  std::vector<double> xq;
  std::vector<int32_t> qlo, qcnt, jst, jw;
  std::vector<double> R[4];
};

int build_rule(int p, int64_t ne, WQRule& W) {
  const std::vector<double> U = open_knots(p, ne);
  const int64_t n = ne + p - 2;
  W.n = n;
  W.NJ = 2 * p + 1;
  std::set<double> pts;
  for (int64_t k = 0; k <= 2 * ne; ++k) pts.insert((double)k / (double)(2 * ne));
  for (int64_t k = 0; k < ne; ++k)
    if (k < p || k >= ne - p) {
      pts.insert((k + 0.25) / (double)ne);
      pts.insert((k + 0.75) / (double)ne);
    }
  W.xq.assign(pts.begin(), pts.end());
  W.nq = (int64_t)W.xq.size();
  std::vector<char> base(W.nq);
  for (int64_t q = 0; q < W.nq; ++q) {
    const double t = W.xq[q] * 2.0 * ne;
    base[q] = std::fabs(t - std::round(t)) < 1e-9;
  }
  // trial values at the points and at Gauss points (p + 2 per element, exact for the moments)
  std::vector<double> E[2];
  for (int b = 0; b < 2; ++b) {
    E[b].assign((size_t)W.nq * n, 0.0);
    for (int64_t q = 0; q < W.nq; ++q) interior_values(p, ne, U, W.xq[q], b, &E[b][q * n]);
  }
  std::vector<double> gx, gw;
  gauss_legendre(p + 2, gx, gw);
  std::vector<double> xg, wg;
  for (int64_t e = 0; e < ne; ++e)
    for (size_t k = 0; k < gx.size(); ++k) {
      const double a = (double)e / ne, b = (double)(e + 1) / ne;
      xg.push_back(0.5 * (a + b) + 0.5 * (b - a) * gx[k]);
      wg.push_back(0.5 * (b - a) * gw[k]);
    }
  std::vector<double> Gv[2];
  for (int b = 0; b < 2; ++b) {
    Gv[b].assign(xg.size() * n, 0.0);
    for (size_t g = 0; g < xg.size(); ++g) interior_values(p, ne, U, xg[g], b, &Gv[b][g * n]);
  }
  W.qlo.assign(n, 0);
  W.qcnt.assign(n, 0);
  W.jst.assign(n, 0);
  W.jw.assign(n, 0);
  for (int64_t i = 0; i < n; ++i) {
    const double lo = U[i + 1], hi = U[i + p + 2];
    int64_t q0 = -1, q1 = -1;
    for (int64_t q = 0; q < W.nq; ++q)
      if (W.xq[q] >= lo - 1e-14 && W.xq[q] <= hi + 1e-14) {
        if (q0 < 0) q0 = q;
        q1 = q;
      }
    W.qlo[i] = (int32_t)q0;
    W.qcnt[i] = (int32_t)(q1 - q0 + 1);
    W.QM = std::max(W.QM, W.qcnt[i]);
    W.jst[i] = (int32_t)std::max<int64_t>(0, i - p);
    W.jw[i] = (int32_t)(std::min<int64_t>(n - 1, i + p) - W.jst[i] + 1);
  }
  for (int ab = 0; ab < 4; ++ab) W.R[ab].assign((size_t)n * W.NJ * W.QM, 0.0);
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 2; ++b)
      for (int64_t i = 0; i < n; ++i) {
        const int nj = W.jw[i];
        std::vector<double> mom(nj, 0.0);
        for (int jj = 0; jj < nj; ++jj) {
          const int64_t j = W.jst[i] + jj;
          double s = 0;
          for (size_t g = 0; g < xg.size(); ++g) s += wg[g] * Gv[a][g * n + i] * Gv[b][g * n + j];
          mom[jj] = s;
        }
        bool ok = false;
        std::vector<double> w;
        std::vector<int64_t> qs;
        for (int pass = 0; pass < 2 && !ok; ++pass) {
          qs.clear();
          for (int64_t q = W.qlo[i]; q < W.qlo[i] + W.qcnt[i]; ++q)
            if (pass == 1 || base[q]) qs.push_back(q);
          std::vector<double> B((size_t)nj * qs.size());
          for (int jj = 0; jj < nj; ++jj)
            for (size_t k = 0; k < qs.size(); ++k) B[jj * qs.size() + k] = E[b][qs[k] * n + W.jst[i] + jj];
          ok = min_norm(B, nj, (int)qs.size(), mom, w);
        }
        FDIGA_CHECK(ok, FDIGA_ERR_INVALID_ARG, "WQ moment system of row %lld not solvable", (long long)i);
        double* R = &W.R[a * 2 + b][(size_t)i * W.NJ * W.QM];
        for (int jj = 0; jj < nj; ++jj)
          for (size_t k = 0; k < qs.size(); ++k)
            R[jj * W.QM + (qs[k] - W.qlo[i])] += w[k] * E[b][qs[k] * n + W.jst[i] + jj];
      }
  return FDIGA_OK;
}

// Q(xi) = det(J) J^{-1} J^{-T} at every point of the tensor grid of the 1D rule: NC = D(D+1)/2 entries
template <int D>
__global__ void wq_coeff_kernel(Geo g, const double* __restrict__ xq, int64_t nq, int64_t q3lo, int64_t q3cnt,
                                double* __restrict__ c) {
  constexpr int NC = D * (D + 1) / 2;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int64_t npts = nq * (D == 3 ? nq * q3cnt : q3cnt);
  if (t >= npts) return;
  const int64_t q1 = t % nq, q2 = (t / nq) % (D == 3 ? nq : q3cnt), q3 = D == 3 ? q3lo + t / (nq * nq) : 0;
  const double x0 = xq[q1], x1 = xq[D == 3 ? q2 : q3lo + q2], x2 = D == 3 ? xq[q3] : 0.0;
  const JH jh = geometry_jh(g, x0, x1, x2);
  double Ji[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Ji[a][b] = 0;
  inv_small<D>(jh.J, Ji);
  double det = jh.J[0][0] * jh.J[1][1] - jh.J[0][1] * jh.J[1][0];
  if (D == 3)
    det = jh.J[0][0] * (jh.J[1][1] * jh.J[2][2] - jh.J[1][2] * jh.J[2][1]) -
          jh.J[0][1] * (jh.J[1][0] * jh.J[2][2] - jh.J[1][2] * jh.J[2][0]) +
          jh.J[0][2] * (jh.J[1][0] * jh.J[2][1] - jh.J[1][1] * jh.J[2][0]);
  int k = 0;
  for (int a = 0; a < D; ++a)
    for (int b = a; b < D; ++b) {
      double s = 0;
      for (int e = 0; e < D; ++e) s += Ji[a][e] * Ji[b][e];
      c[t * NC + k++] = det * s;
    }
}

struct WqRowArgs {
  int64_t n, nq, row0, nrows, q3lo;  // q3lo: first point of the local coefficient slab (3D)
  int NJ, QM;
  const int32_t *qlo, *qcnt, *jst, *jw;
  const double* R[4];
  const double* c;
  const int64_t *pre1, *pre2, *pre3;
  int64_t S1, S2, vbase;
  double* vals;  // canonical layout, zeroed
};

__device__ __forceinline__ int qidx(int a, int b, int D) {  // position of Q_ab (a <= b) in the packed NC
  if (a > b) {
    const int t = a;
    a = b;
    b = t;
  }
  return D == 2 ? (a == 0 ? b : 2) : (a == 0 ? b : (a == 1 ? 2 + b : 5));
}

template <int D>
__global__ void wq_row_kernel(WqRowArgs A) {
  constexpr int NC = D * (D + 1) / 2;
  constexpr int JM = 11;  // window bound (p <= 5)
  const int64_t lr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lr >= A.nrows) return;
  const int64_t row = A.row0 + lr;
  const int64_t n = A.n;
  const int64_t i1 = row % n, i2 = (row / n) % n, i3 = D == 3 ? row / (n * n) : 0;
  const int w1 = A.jw[i1], w2 = A.jw[i2], w3 = D == 3 ? A.jw[i3] : 1;
  const int c1 = A.qcnt[i1], c2 = A.qcnt[i2], c3 = D == 3 ? A.qcnt[i3] : 1;
  const int64_t o1 = A.qlo[i1], o2 = A.qlo[i2], o3 = D == 3 ? A.qlo[i3] - A.q3lo : 0;
  const int64_t nq = A.nq;
  // canonical row offset (rows in flattened order, each with its w3 w2 w1 box, j1 fastest)
  const int64_t cb = (D == 3 ? A.pre3[i3] * A.S2 * A.S1 : 0) + (int64_t)w3 * A.pre2[i2] * A.S1 +
                     (int64_t)w3 * w2 * A.pre1[i1] - A.vbase;
  double* out = A.vals + cb;
  double v[JM], acc2[JM * JM];
  for (int al = 0; al < D; ++al)
    for (int be = 0; be < D; ++be) {
      const int comp = qidx(al, be, D);
      const double* R1 = A.R[(al == 0) * 2 + (be == 0)] + i1 * A.NJ * A.QM;
      const double* R2 = A.R[(al == 1) * 2 + (be == 1)] + i2 * A.NJ * A.QM;
      const double* R3 = D == 3 ? A.R[(al == 2) * 2 + (be == 2)] + i3 * A.NJ * A.QM : nullptr;
      for (int q3 = 0; q3 < c3; ++q3) {
        for (int k = 0; k < w2 * w1; ++k) acc2[k] = 0.0;
        for (int q2 = 0; q2 < c2; ++q2) {
          const double* cq = A.c + (((o3 + q3) * (D == 3 ? nq : 0) + (o2 + q2)) * nq + o1) * NC + comp;
          for (int j1 = 0; j1 < w1; ++j1) {
            double s = 0;
            for (int q1 = 0; q1 < c1; ++q1) s = fma(R1[j1 * A.QM + q1], cq[q1 * NC], s);
            v[j1] = s;
          }
          for (int j2 = 0; j2 < w2; ++j2) {
            const double r2 = R2[j2 * A.QM + q2];
            for (int j1 = 0; j1 < w1; ++j1) acc2[j2 * w1 + j1] = fma(r2, v[j1], acc2[j2 * w1 + j1]);
          }
        }
        for (int j3 = 0; j3 < w3; ++j3) {
          const double r3 = D == 3 ? R3[j3 * A.QM + q3] : 1.0;
          for (int k = 0; k < w2 * w1; ++k) out[j3 * w2 * w1 + k] = fma(r3, acc2[k], out[j3 * w2 * w1 + k]);
        }
      }
    }
}

}  // namespace

extern "C" {

int galerkin_1d_factors(int p, int64_t ne, double* M, double* K) {
  FDIGA_CHECK(M && K && p >= 1 && ne >= 1 && ne + p - 2 >= 1, FDIGA_ERR_INVALID_ARG,
              "bad galerkin_1d_factors arguments");
  const std::vector<double> U = open_knots(p, ne);
  const int64_t n = ne + p - 2;
  std::vector<double> gx, gw;
  gauss_legendre(p + 2, gx, gw);
  std::memset(M, 0, n * n * sizeof(double));
  std::memset(K, 0, n * n * sizeof(double));
  std::vector<double> b0(n), b1(n);
  for (int64_t e = 0; e < ne; ++e)
    for (size_t k = 0; k < gx.size(); ++k) {
      const double a = (double)e / ne, b = (double)(e + 1) / ne;
      const double x = 0.5 * (a + b) + 0.5 * (b - a) * gx[k], w = 0.5 * (b - a) * gw[k];
      interior_values(p, ne, U, x, 0, b0.data());
      interior_values(p, ne, U, x, 1, b1.data());
      for (int64_t i = 0; i < n; ++i) {
        if (b0[i] == 0.0 && b1[i] == 0.0) continue;
        for (int64_t j = 0; j < n; ++j) {
          M[i * n + j] += w * b0[i] * b0[j];
          K[i * n + j] += w * b1[i] * b1[j];
        }
      }
    }
  return FDIGA_OK;
}

// stencil_create is the common tail (stencil.cu)
int wq_assemble(fdiga_ctx* ctx, int d, int p, int64_t ne, int geometry_id, const double* geo_params,
                fdiga_stencil** out) {
  FDIGA_CHECK(ctx && out, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_CHECK(d == 2 || d == 3, FDIGA_ERR_INVALID_ARG, "d must be 2 or 3");
  FDIGA_CHECK(p >= 1 && p <= 5 && ne >= 1 && ne + p - 2 >= 1, FDIGA_ERR_INVALID_ARG, "p = %d, ne = %lld", p,
              (long long)ne);
  const bool ok_geo = geometry_id == FDIGA_GEOM_IDENTITY || (geometry_id == FDIGA_GEOM_ANNULUS && d == 2) ||
                      ((geometry_id == FDIGA_GEOM_DEFORMED_CUBE || geometry_id == FDIGA_GEOM_THICK_RING) && d == 3);
  FDIGA_CHECK(ok_geo, FDIGA_ERR_INVALID_ARG, "geometry %d not available in %dD", geometry_id, d);
  FDIGA_CHECK(!ctx->sharded || d == 3, FDIGA_ERR_NOT_SUPPORTED, "2D operators are not sharded (replicas only)");
  FDIGA_TRY(bind(ctx));
  WQRule W;
  FDIGA_TRY(build_rule(p, ne, W));
  const int64_t n = W.n;
  Geo g{};
  g.id = geometry_id;
  const int np = geometry_id == FDIGA_GEOM_ANNULUS ? 2 : geometry_id == FDIGA_GEOM_DEFORMED_CUBE ? 1
                                                       : geometry_id == FDIGA_GEOM_THICK_RING  ? 3 : 0;
  FDIGA_CHECK(np == 0 || geo_params, FDIGA_ERR_INVALID_ARG, "geometry %d needs %d parameters", geometry_id, np);
  for (int k = 0; k < np; ++k) g.prm[k] = geo_params[k];
  // local rows (slab of the last axis) and the window structure of the tensor-window layout
  int64_t o = 0, e = n;
  partition(n, ctx->sharded ? ctx->nranks : 1, ctx->sharded ? ctx->rank : 0, &o, &e);
  if (d == 2) {
    o = 0;
    e = n;
  }
  std::vector<int64_t> pre(n + 1, 0);
  for (int64_t i = 0; i < n; ++i) pre[i + 1] = pre[i] + W.jw[i];
  const int64_t S = pre[n];
  const int64_t vbase = d == 3 ? pre[o] * S * S : 0;
  const int64_t nloc = d == 3 ? (pre[e] - pre[o]) * S * S : S * S;
  // points of the local coefficient slab along direction 3
  int64_t q3lo = 0, q3hi = W.nq;
  if (d == 3 && e > o) {
    q3lo = W.qlo[o];
    q3hi = 0;
    for (int64_t i = o; i < e; ++i) q3hi = std::max<int64_t>(q3hi, W.qlo[i] + W.qcnt[i]);
  }
  const int NC = d * (d + 1) / 2;
  const int64_t npts = W.nq * (d == 3 ? W.nq * (q3hi - q3lo) : (q3hi - q3lo));
  std::vector<void*> tmp;
  auto upload = [&](const void* h, size_t bytes) -> void* {
    void* dptr = nullptr;
    if (cudaMalloc(&dptr, std::max<size_t>(bytes, 8)) != cudaSuccess) return nullptr;
    tmp.push_back(dptr);
    if (bytes && h) cudaMemcpy(dptr, h, bytes, cudaMemcpyHostToDevice);
    return dptr;
  };
  int s = FDIGA_OK;
  WqRowArgs A{};
  A.n = n;
  A.nq = W.nq;
  A.NJ = W.NJ;
  A.QM = W.QM;
  A.q3lo = q3lo;
  A.qlo = (const int32_t*)upload(W.qlo.data(), n * 4);
  A.qcnt = (const int32_t*)upload(W.qcnt.data(), n * 4);
  A.jst = (const int32_t*)upload(W.jst.data(), n * 4);
  A.jw = (const int32_t*)upload(W.jw.data(), n * 4);
  for (int ab = 0; ab < 4; ++ab) A.R[ab] = (const double*)upload(W.R[ab].data(), W.R[ab].size() * 8);
  const double* dxq = (const double*)upload(W.xq.data(), W.nq * 8);
  A.pre1 = A.pre2 = A.pre3 = (const int64_t*)upload(pre.data(), (n + 1) * 8);
  A.S1 = S;
  A.S2 = S;
  A.vbase = vbase;
  A.row0 = d == 3 ? o * n * n : 0;
  A.nrows = d == 3 ? (e - o) * n * n : n * n;
  double* c = (double*)upload(nullptr, npts * NC * 8);
  double* vals = (double*)upload(nullptr, nloc * 8);
  for (void* q : tmp)
    if (!q) s = FDIGA_ERR_OOM;
  if (s == FDIGA_OK) {
    A.c = c;
    A.vals = vals;
    cudaStream_t st = ctx->stream;
    if (npts) {
      if (d == 3)
        wq_coeff_kernel<3><<<(unsigned)((npts + 127) / 128), 128, 0, st>>>(g, dxq, W.nq, q3lo, q3hi - q3lo, c);
      else
        wq_coeff_kernel<2><<<(unsigned)((npts + 127) / 128), 128, 0, st>>>(g, dxq, W.nq, 0, W.nq, c);
      count_launch(ctx);
    }
    cudaMemsetAsync(vals, 0, nloc * 8, st);
    if (A.nrows) {
      if (d == 3)
        wq_row_kernel<3><<<(unsigned)((A.nrows + 127) / 128), 128, 0, st>>>(A);
      else
        wq_row_kernel<2><<<(unsigned)((A.nrows + 127) / 128), 128, 0, st>>>(A);
      count_launch(ctx);
    }
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess) err = cudaStreamSynchronize(st);
    if (err != cudaSuccess) {
      set_error("wq_assemble: %s", cudaGetErrorString(err));
      s = FDIGA_ERR_CUDA;
    }
  }
  if (s == FDIGA_OK) {
    const int64_t nn[3] = {n, n, n};
    const int32_t* st3[3] = {W.jst.data(), W.jst.data(), W.jst.data()};
    const int32_t* wd3[3] = {W.jw.data(), W.jw.data(), W.jw.data()};
    s = stencil_create(ctx, d, nn, st3, wd3, vals, 1, out);
  }
  for (void* q : tmp) cudaFree(q);
  return s;
}

}  // extern "C"

// Collocation operator A_C: device assembly on analytic geometries and the stored-operator matvec.
//
// Row i = tau_i (Greville point) of eq:collocation:
//   (A_C)_{ij} = -Lap_x (B^_j o F^{-1})(F(tau_i)),  K = I.
// With x = F(xi), J = dF/dxi, H_c = d^2 F_c/dxi^2 (chain rule):
//   A_ij = - sum_{a,b} G_ab d_a d_b B^_j(tau_i) + sum_a beta_a d_a B^_j(tau_i),
//   G = (J^T J)^{-1},  beta_a = sum_c (J^{-1})_{ac} tr(G H_c),
// and d^t B^_j(tau_i) = prod_l B_{j_l}^{(t_l)}(tau_{l,i_l}) (tensor-product basis).
//
// Storage ("tensor window"): per direction l and 1D index i, the contiguous column window
// [start_l(i), start_l(i) + width_l(i)) holding every interior basis function whose value or first
// two derivatives at tau_{l,i} is nonzero.  Row i stores the w_3 w_2 w_1 values of its column box
// (j_1 fastest); row offsets follow from prefix sums of the widths, so no index arrays are stored
// and the matvec moves exactly 8 nnz + 16 N bytes.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "geometry.cuh"
#include "bspline.h"
#include "matfree.cuh"

using namespace fdiga;

struct fdiga_stencil {
  fdiga_ctx* ctx = nullptr;
  int d = 0;
  int64_t n[3] = {1, 1, 1};      // direction sizes (n[2] = 1 in 2D)
  int64_t N = 0, nnz = 0;
  int wmax = 0;                   // max window width over all directions
  std::vector<int32_t> hstart[3], hwidth[3];
  std::vector<int64_t> hpre[3];   // prefix sums of widths, length n+1
  int32_t* start[3] = {nullptr, nullptr, nullptr};
  int32_t* width[3] = {nullptr, nullptr, nullptr};
  int64_t* pre[3] = {nullptr, nullptr, nullptr};
  double* vals = nullptr;         // nnz values, INTERNAL layout (see below)
  // internal "line-SoA" layout: the values of line (i3, i2) occupy the same range as in the canonical
  // layout, ordered [q = a*w2 + b][c][i1 among the rows of the line with w1(i1) > c], so a warp of
  // consecutive rows reads consecutive addresses for every (q, c).  voff1[i1 * wm1 + c] is the offset
  // of (i1, c) inside one q-block of S1 values.
  int wm1 = 0;                    // max window width in direction 1
  int32_t* voff1 = nullptr;       // device, n1 x wm1
  std::vector<int32_t> hvoff1;
  // slab sharding of the rows (3D, nranks > 1): this rank stores the rows of planes
  // i3 in [o, e) (Nloc rows, values from offset vbase of the global layout on) and reads x planes
  // [lo, hi); the planes outside [o, e) arrive from their owners into halo_lo / halo_hi.
  int64_t o = 0, e = 1, lo = 0, hi = 1, Nloc = 0, vbase = 0;
  double* halo = nullptr;         // (o - lo + hi - e) planes: lower halo, then upper halo
  std::vector<fdiga::P2PMsg> hsend, hrecv;  // halo messages (x pointers patched per call)
  std::vector<int64_t> hsend_plane;         // first plane (global) of each send
  // matrix-free operator (NEXT-1, matfree.cu): no stored values; 1D tables and the map on the device
  bool mf = false;
  int mf_W = 0, mf_B[3] = {0, 0, 0};
  double* mf_tau[3] = {nullptr, nullptr, nullptr};
  double* mf_tab[3] = {nullptr, nullptr, nullptr};
  double* mf_trig[3] = {nullptr, nullptr, nullptr};  // (sin, cos)(theta tau) per direction
  int32_t* mf_box[3] = {nullptr, nullptr, nullptr};  // per tile: (first column, extent) of its x box
  fdiga::Geo mf_geo{};
};

namespace {

// 1D tables for one direction: Greville points, windows, and B^{(r)}_j(tau_i) on the window.
struct Table1D {
  int64_t n = 0;
  int wmax = 0;
  std::vector<double> tau;
  std::vector<int32_t> start, width;
  std::vector<double> val[3];  // val[r][i * wmax + c] = B^{(r)}_{start(i)+c}(tau_i)
};

void build_table(int p, int64_t ne, Table1D& T) {
  const int64_t m = ne + p;  // number of basis functions
  const int64_t n = m - 2;
  std::vector<double> U;
  for (int k = 0; k <= p; ++k) U.push_back(0.0);
  for (int64_t k = 1; k < ne; ++k) U.push_back((double)k / (double)ne);
  for (int k = 0; k <= p; ++k) U.push_back(1.0);
  T.n = n;
  T.wmax = p + 1;
  T.tau.resize(n);
  T.start.resize(n);
  T.width.resize(n);
  for (int r = 0; r < 3; ++r) T.val[r].assign(n * T.wmax, 0.0);
  for (int64_t i = 1; i <= n; ++i) {  // interior function i (0-based full index), Greville point of P:164
    double s = 0;
    for (int j = 1; j <= p; ++j) s += U[i + j];
    const double t = s / p;
    T.tau[i - 1] = t;
    // knot span: U[span] <= t < U[span+1], span in [p, m-1]
    int span = p;
    while (span < m - 1 && U[span + 1] <= t) ++span;
    std::vector<std::vector<double>> ders;
    ders_basis_funs(span, t, p, std::min(2, p), U, ders);
    while ((int)ders.size() < 3) ders.push_back(std::vector<double>(p + 1, 0.0));
    // window: first/last full index among span-p..span with a nonzero value or 1st/2nd derivative,
    // clipped to the interior functions 1..m-2
    int64_t first = -1, last = -1;
    for (int r = 0; r <= p; ++r) {
      const int64_t k = span - p + r;
      if (k < 1 || k > m - 2) continue;
      if (ders[0][r] != 0.0 || ders[1][r] != 0.0 || ders[2][r] != 0.0) {
        if (first < 0) first = k;
        last = k;
      }
    }
    T.start[i - 1] = (int32_t)(first - 1);
    T.width[i - 1] = (int32_t)(last - first + 1);
    for (int64_t k = first; k <= last; ++k) {
      const int r = (int)(k - (span - p));
      for (int q = 0; q < 3; ++q) T.val[q][(i - 1) * T.wmax + (k - first)] = ders[q][r];
    }
  }
}

struct AsmArgs {
  int wmax;
  int64_t n1, n2, n3, S1, S2;
  const double *tau1, *tau2, *tau3;
  const int32_t *w1, *w2, *w3;
  const int64_t *pre1, *pre2, *pre3;
  const double *tab1, *tab2, *tab3;  // tab_l[(r * n_l + i) * wmax + c] = B^{(r)}_{start_l(i)+c}(tau_{l,i})
  const int32_t* voff1;              // internal layout offsets (n1 x wm1)
  int wm1;
  Geo geo;
  double* vals;
  int64_t row0, nrows, vbase;  // sharded: global row of thread 0, rows to assemble, value offset of row0
};

// One thread per collocation row: geometry coefficients G = (J^T J)^{-1}, beta, then the w3*w2*w1
// box of values  sum_t c_t prod_l B^{(t_l)}.  All small arrays are statically indexed (registers).
template <int D>
__global__ void assemble_kernel(AsmArgs A) {
  const int64_t lrow = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lrow >= A.nrows) return;
  const int64_t row = A.row0 + lrow;
  const int64_t i1 = row % A.n1, i2 = (row / A.n1) % A.n2, i3 = row / (A.n1 * A.n2);
  const double x0 = A.tau1[i1], x1 = A.tau2[i2], x2 = (D == 3) ? A.tau3[i3] : 0.0;
  double G[3][3], beta[3];
  {
    const double th = geo_theta(A.geo.id);
    double sn[3], cs[3];
    sincos(th * x0, &sn[0], &cs[0]);
    sincos(th * x1, &sn[1], &cs[1]);
    sincos(th * x2, &sn[2], &cs[2]);
    double F[3], w[3];
    geometry_F(A.geo, x0, x1, x2, sn, cs, F);
    wind_at(A.geo, F, w);
    colloc_coeffs<D>(geometry_jh(A.geo, x0, sn, cs), G, beta, A.geo.wind ? w : nullptr);
  }
  const int W = A.wmax;
  const int w1 = A.w1[i1];
  const int w2 = A.w2[i2];
  const int w3 = (D == 3) ? A.w3[i3] : 1;
  const int64_t line = (D == 3 ? A.pre3[i3] * A.S2 * A.S1 : 0) + (int64_t)w3 * A.pre2[i2] * A.S1;
  const int32_t* vo = A.voff1 + i1 * A.wm1;
  // 1D factor rows at this point: f_l[r] = &tab_l[(r n_l + i_l) W]
  const double* f1[3];
  const double* f2[3];
  const double* f3[3];
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    f1[r] = A.tab1 + (r * A.n1 + i1) * W;
    f2[r] = A.tab2 + (r * A.n2 + i2) * W;
    f3[r] = (D == 3) ? A.tab3 + (r * A.n3 + i3) * W : nullptr;
  }
  double* out = A.vals + (line - A.vbase);
  for (int a = 0; a < w3; ++a)
    for (int b = 0; b < w2; ++b)
      for (int c = 0; c < w1; ++c) {
        double v = 0;
        // -G_ab d_a d_b  (t = e_a + e_b) and beta_a d_a  (t = e_a)
#pragma unroll
        for (int p = 0; p < D; ++p)
#pragma unroll
          for (int q = 0; q < D; ++q) {
            const int t1 = (p == 0) + (q == 0), t2 = (p == 1) + (q == 1), t3 = (p == 2) + (q == 2);
            double prod = -G[p][q] * f1[t1][c] * f2[t2][b];
            if (D == 3) prod *= f3[t3][a];
            v += prod;
          }
#pragma unroll
        for (int p = 0; p < D; ++p) {
          const int t1 = (p == 0), t2 = (p == 1), t3 = (p == 2);
          double prod = beta[p] * f1[t1][c] * f2[t2][b];
          if (D == 3) prod *= f3[t3][a];
          v += prod;
        }
        out[((int64_t)a * w2 + b) * A.S1 + vo[c]] = v;
      }
}

// ------------------------------------------------------------------ matvec
struct MvArgs {
  int64_t n1, n2, n3, N, S1, S2;
  const int32_t *st1, *st2, *st3, *w1, *w2, *w3;
  const int64_t *pre2, *pre3;
  const int32_t* voff1;
  const double* vals;
  const double* x;
  double* y;
  const int* skip;  // device flag: nonzero -> no-op (GMRES graph early exit)
  // sharded rows (SH = true): local row r is global row r + o n1 n2; x holds planes [o, e), halo_lo
  // planes [lo, o), halo_hi planes [e, hi)
  int64_t o, e, lo, vbase;
  const double *halo_lo, *halo_hi;
};

template <bool SH>
__device__ __forceinline__ const double* x_plane(const MvArgs& A, int64_t g, int64_t n12) {
  if (!SH) return A.x + g * n12;
  if (g < A.o) return A.halo_lo + (g - A.lo) * n12;
  if (g >= A.e) return A.halo_hi + (g - A.e) * n12;
  return A.x + (g - A.o) * n12;
}

// y = A x, one thread per row (flattened, i1 fastest).  For every window pair q = (a, b) the thread
// reads its w1 <= WM values at vals[line + q S1 + voff1(i1, c)] -- consecutive rows hit consecutive
// addresses, so every warp load is a full 256-byte coalesced stream (values are read exactly once,
// streaming / evict-first) -- and the matching x window x[(s3+a) n1 n2 + (s2+b) n1 + s1 + c]
// through L1/L2 (x of neighbouring rows overlaps).  Bytes moved: 8 nnz + 16 N.
template <int WM, int UB, int MINB, bool SH>
__global__ void __launch_bounds__(256, MINB) matvec_kernel(MvArgs A) {
  const uint32_t r = blockIdx.x * 256u + threadIdx.x;
  if (r >= (uint32_t)A.N || (A.skip && *A.skip)) return;
  const uint32_t n1 = (uint32_t)A.n1, n2 = (uint32_t)A.n2;
  const uint32_t i1 = r % n1, line = r / n1;
  const uint32_t i2 = line % n2, i3 = line / n2 + (SH ? (uint32_t)A.o : 0u);
  const int w1 = __ldg(A.w1 + i1), w2 = __ldg(A.w2 + i2), w3 = __ldg(A.w3 + i3);
  const int64_t S1 = A.S1;
  const int64_t n12 = (int64_t)n1 * n2;
  // per-thread value pointers for every column c of the window; advanced by UB * S1 per batch of
  // UB window pairs q = a * w2 + b
  const double* __restrict__ vbase =
      A.vals + (__ldg(A.pre3 + i3) * A.S2 * S1 - (SH ? A.vbase : 0)) + (int64_t)w3 * __ldg(A.pre2 + i2) * S1;
  const double* pv[WM];
#pragma unroll
  for (int c = 0; c < WM; ++c) pv[c] = vbase + ((c < w1) ? __ldg(A.voff1 + i1 * WM + c) : 0);
  const int64_t g0 = __ldg(A.st3 + i3);
  const int64_t xoff = (int64_t)__ldg(A.st2 + i2) * n1 + __ldg(A.st1 + i1);
  const double* __restrict__ xa = x_plane<SH>(A, g0, n12) + xoff;  // x window row of plane g0 + a
  const int nq = w3 * w2;
  int a = 0, b = 0;
  double acc[UB];
#pragma unroll
  for (int u = 0; u < UB; ++u) acc[u] = 0.0;
  for (int q0 = 0; q0 < nq; q0 += UB) {
    // issue every value load of the batch first (memory-level parallelism), then the x loads + FMAs
    double vv[UB][WM];
#pragma unroll
    for (int u = 0; u < UB; ++u)
#pragma unroll
      for (int c = 0; c < WM; ++c) vv[u][c] = (q0 + u < nq && c < w1) ? __ldcs(pv[c] + u * S1) : 0.0;
#pragma unroll
    for (int u = 0; u < UB; ++u) {
      if (q0 + u < nq) {
        const double* xq = xa + (int64_t)b * n1;
#pragma unroll
        for (int c = 0; c < WM; ++c)
          if (c < w1) acc[u] = fma(vv[u][c], __ldg(xq + c), acc[u]);
        if (++b == w2) {
          b = 0;
          ++a;
          xa = x_plane<SH>(A, g0 + a, n12) + xoff;
        }
      }
    }
#pragma unroll
    for (int c = 0; c < WM; ++c) pv[c] += UB * S1;
  }
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < UB; ++u) s += acc[u];
  A.y[r] = s;
}

// canonical <-> internal value layouts (one thread per row)
struct PermArgs {
  int64_t n1, n2, n3, N, S1, S2;
  const int32_t *w1, *w2, *w3;
  const int64_t *pre1, *pre2, *pre3;
  const int32_t* voff1;
  int wm1;
  const double* src;
  double* dst;
  int to_internal;
  int64_t row0, vbase;  // sharded: first global row, value offset of that row (P.N = local rows)
};

__global__ void permute_kernel(PermArgs P) {
  const int64_t lr = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (lr >= P.N) return;
  const int64_t r = P.row0 + lr;
  const int64_t i1 = r % P.n1, line = r / P.n1;
  const int64_t i2 = line % P.n2, i3 = line / P.n2;
  const int w1 = P.w1[i1], w2 = P.w2[i2], w3 = P.w3[i3];
  const int64_t lb = P.pre3[i3] * P.S2 * P.S1 + (int64_t)w3 * P.pre2[i2] * P.S1 - P.vbase;
  const int64_t cb = lb + (int64_t)w3 * w2 * P.pre1[i1];
  for (int q = 0; q < w3 * w2; ++q)
    for (int c = 0; c < w1; ++c) {
      const int64_t ci = cb + (int64_t)q * w1 + c;
      const int64_t ii = lb + (int64_t)q * P.S1 + P.voff1[i1 * P.wm1 + c];
      if (P.to_internal) P.dst[ii] = P.src[ci];
      else P.dst[ci] = P.src[ii];
    }
}

MvArgs make_mv_args(const fdiga_stencil* S, const double* x, double* y) {
  MvArgs A{};
  A.n1 = S->n[0];
  A.n2 = S->n[1];
  A.n3 = S->n[2];
  A.N = S->Nloc;
  A.S1 = S->hpre[0][S->n[0]];
  A.S2 = S->hpre[1][S->n[1]];
  A.o = S->o;
  A.e = S->e;
  A.lo = S->lo;
  A.vbase = S->vbase;
  const int64_t plane = S->n[0] * S->n[1];
  A.halo_lo = S->halo;
  A.halo_hi = S->halo ? S->halo + (S->o - S->lo) * plane : nullptr;
  A.st1 = S->start[0];
  A.st2 = S->start[1];
  A.st3 = S->start[2];
  A.w1 = S->width[0];
  A.w2 = S->width[1];
  A.w3 = S->width[2];
  A.pre2 = S->pre[1];
  A.pre3 = S->pre[2];
  A.voff1 = S->voff1;
  A.vals = S->vals;
  A.x = x;
  A.y = y;
  return A;
}

int permute_values(fdiga_stencil* S, const double* src, double* dst, int to_internal) {
  PermArgs P{};
  P.n1 = S->n[0];
  P.n2 = S->n[1];
  P.n3 = S->n[2];
  P.N = S->Nloc;
  P.row0 = S->o * S->n[0] * S->n[1];
  P.vbase = S->vbase;
  P.S1 = S->hpre[0][S->n[0]];
  P.S2 = S->hpre[1][S->n[1]];
  P.w1 = S->width[0];
  P.w2 = S->width[1];
  P.w3 = S->width[2];
  P.pre1 = S->pre[0];
  P.pre2 = S->pre[1];
  P.pre3 = S->pre[2];
  P.voff1 = S->voff1;
  P.wm1 = S->wm1;
  P.src = src;
  P.dst = dst;
  P.to_internal = to_internal;
  if (S->Nloc == 0) return FDIGA_OK;
  permute_kernel<<<(unsigned)((S->Nloc + 255) / 256), 256, 0, S->ctx->stream>>>(P);
  count_launch(S->ctx);
  FDIGA_CUDA(cudaGetLastError());
  FDIGA_CUDA(cudaStreamSynchronize(S->ctx->stream));
  return FDIGA_OK;
}

// Common tail of stencil_create / colloc_assemble: tables on the device, internal-layout offsets.
int finish_stencil(fdiga_stencil* S) {
  for (int l = 0; l < 3; ++l) {
    const int64_t nl = S->n[l];
    S->hpre[l].assign(nl + 1, 0);
    for (int64_t i = 0; i < nl; ++i) {
      FDIGA_CHECK(S->hwidth[l][i] >= 1 && S->hstart[l][i] >= 0 && S->hstart[l][i] + S->hwidth[l][i] <= nl,
                  FDIGA_ERR_INVALID_ARG, "bad window in direction %d at %lld", l, (long long)i);
      S->hpre[l][i + 1] = S->hpre[l][i] + S->hwidth[l][i];
      S->wmax = std::max<int>(S->wmax, S->hwidth[l][i]);
    }
    FDIGA_CUDA(cudaMalloc(&S->start[l], nl * sizeof(int32_t)));
    FDIGA_CUDA(cudaMalloc(&S->width[l], nl * sizeof(int32_t)));
    FDIGA_CUDA(cudaMalloc(&S->pre[l], (nl + 1) * sizeof(int64_t)));
    FDIGA_CUDA(cudaMemcpy(S->start[l], S->hstart[l].data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice));
    FDIGA_CUDA(cudaMemcpy(S->width[l], S->hwidth[l].data(), nl * sizeof(int32_t), cudaMemcpyHostToDevice));
    FDIGA_CUDA(cudaMemcpy(S->pre[l], S->hpre[l].data(), (nl + 1) * sizeof(int64_t), cudaMemcpyHostToDevice));
  }
  // this rank's slab of planes (3D) and the x planes its rows read
  fdiga_ctx* ctx = S->ctx;
  const int64_t plane = S->n[0] * S->n[1];
  partition(S->n[2], ctx->nranks, ctx->rank, &S->o, &S->e);
  S->Nloc = (S->e - S->o) * plane;
  const int64_t S12 = S->hpre[0][S->n[0]] * S->hpre[1][S->n[1]];
  S->vbase = S->hpre[2][S->o] * S12;
  S->nnz = (S->hpre[2][S->e] - S->hpre[2][S->o]) * S12;
  const int nr = ctx->sharded ? ctx->nranks : 1;
  std::vector<int64_t> sb(nr), se(nr), rb(nr), re(nr);
  FDIGA_TRY(fdiga_halo_plan(S->n[2], S->hstart[2].data(), S->hwidth[2].data(), nr, ctx->sharded ? ctx->rank : 0,
                            &S->lo, &S->hi, sb.data(), se.data(), rb.data(), re.data()));
  if (ctx->sharded) {
    // halo messages: my planes inside every other rank's needed range (one contiguous run per pair)
    S->hsend.clear();
    S->hrecv.clear();
    S->hsend_plane.clear();
    for (int q = 0; q < nr; ++q) {
      if (se[q] > sb[q]) {
        S->hsend.push_back({q, nullptr, (size_t)((se[q] - sb[q]) * plane) * 8});
        S->hsend_plane.push_back(sb[q]);
      }
      if (re[q] > rb[q]) S->hrecv.push_back({q, (void*)(intptr_t)rb[q], (size_t)((re[q] - rb[q]) * plane) * 8});
    }
    const int64_t nh = (S->o - S->lo) + (S->hi - S->e);
    if (nh > 0) {
      FDIGA_CUDA(cudaMalloc(&S->halo, (size_t)nh * plane * sizeof(double)));
      for (auto& m : S->hrecv) {  // patch the destinations: lower halo [lo, o), upper halo [e, hi)
        const int64_t pl = (int64_t)(intptr_t)m.ptr;
        const int64_t off = pl < S->o ? (pl - S->lo) : (S->o - S->lo) + (pl - S->e);
        m.ptr = S->halo + off * plane;
      }
    }
  }
  FDIGA_CHECK(S->hpre[0][S->n[0]] < (int64_t(1) << 31), FDIGA_ERR_NOT_SUPPORTED, "direction-1 windows too large");
  FDIGA_CHECK(S->Nloc < (int64_t(1) << 31) - 256, FDIGA_ERR_NOT_SUPPORTED, "more than 2^31 rows per rank");
  // internal layout: column-major over c within each q-block, rows of the line compacted per column
  const int64_t n1 = S->n[0];
  int wm1 = 0;
  for (int64_t i = 0; i < n1; ++i) wm1 = std::max<int>(wm1, S->hwidth[0][i]);
  FDIGA_CHECK(wm1 <= 11, FDIGA_ERR_NOT_SUPPORTED, "direction-1 window width %d > 11", wm1);
  S->wm1 = wm1;
  S->hvoff1.assign(n1 * wm1, 0);
  int64_t colpre = 0;
  for (int c = 0; c < wm1; ++c) {
    int64_t rank = 0;
    for (int64_t i = 0; i < n1; ++i)
      if (S->hwidth[0][i] > c) S->hvoff1[i * wm1 + c] = (int32_t)(colpre + rank++);
    colpre += rank;
  }
  FDIGA_CUDA(cudaMalloc(&S->voff1, S->hvoff1.size() * sizeof(int32_t)));
  FDIGA_CUDA(cudaMemcpy(S->voff1, S->hvoff1.data(), S->hvoff1.size() * sizeof(int32_t), cudaMemcpyHostToDevice));
  FDIGA_CUDA(cudaDeviceSynchronize());
  return FDIGA_OK;
}

fdiga_stencil* new_stencil(fdiga_ctx* ctx, int d, const int64_t* n) {
  fdiga_stencil* S = new fdiga_stencil();
  S->ctx = ctx;
  S->d = d;
  S->N = 1;
  for (int l = 0; l < 3; ++l) {
    S->n[l] = l < d ? n[l] : 1;
    S->N *= S->n[l];
  }
  if (d == 2) {  // dummy third direction: one plane, window {0}
    S->hstart[2].assign(1, 0);
    S->hwidth[2].assign(1, 1);
  }
  return S;
}

}  // namespace

extern "C" {

int stencil_destroy(fdiga_stencil* S) {
  if (!S) return FDIGA_OK;
  cudaSetDevice(S->ctx->device);
  destroy_gmres_graph(S->ctx);
  for (int l = 0; l < 3; ++l) {
    cudaFree(S->start[l]);
    cudaFree(S->width[l]);
    cudaFree(S->pre[l]);
  }
  cudaFree(S->vals);
  cudaFree(S->voff1);
  cudaFree(S->halo);
  for (int l = 0; l < 3; ++l) {
    cudaFree(S->mf_tau[l]);
    cudaFree(S->mf_tab[l]);
    cudaFree(S->mf_trig[l]);
    cudaFree(S->mf_box[l]);
  }
  delete S;
  return FDIGA_OK;
}

int stencil_create(fdiga_ctx* ctx, int d, const int64_t* n, const int32_t* const* start, const int32_t* const* width,
                   const double* values, int values_on_device, fdiga_stencil** out) {
  FDIGA_CHECK(ctx && n && start && width && values && out, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_CHECK(d == 2 || d == 3, FDIGA_ERR_INVALID_ARG, "d must be 2 or 3");
  FDIGA_CHECK(!ctx->sharded || d == 3, FDIGA_ERR_NOT_SUPPORTED, "2D operators are not sharded (replicas only)");
  *out = nullptr;
  FDIGA_TRY(bind(ctx));
  fdiga_stencil* S = new_stencil(ctx, d, n);
  for (int l = 0; l < d; ++l) {
    S->hstart[l].assign(start[l], start[l] + n[l]);
    S->hwidth[l].assign(width[l], width[l] + n[l]);
  }
  int s = finish_stencil(S);
  double* canon = nullptr;
  if (s == FDIGA_OK) {
    cudaError_t e = cudaMalloc(&S->vals, (S->nnz + 2) * sizeof(double));
    if (e == cudaSuccess) e = cudaMalloc(&canon, S->nnz * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(canon, values, S->nnz * sizeof(double),
                     values_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      set_error("stencil_create: %s", cudaGetErrorString(e));
      s = FDIGA_ERR_CUDA;
    }
  }
  if (s == FDIGA_OK) s = permute_values(S, canon, S->vals, 1);
  cudaFree(canon);
  if (s != FDIGA_OK) {
    stencil_destroy(S);
    return s;
  }
  *out = S;
  return FDIGA_OK;
}

static int colloc_build(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                        int wind_id, const double* wind_params, int matrix_free, fdiga_stencil** out) {
  FDIGA_CHECK(ctx && ne && out, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_CHECK(d == 2 || d == 3, FDIGA_ERR_INVALID_ARG, "d must be 2 or 3");
  FDIGA_CHECK(p >= 1 && p <= 8, FDIGA_ERR_INVALID_ARG, "degree p = %d out of range", p);
  FDIGA_CHECK(!ctx->sharded || d == 3, FDIGA_ERR_NOT_SUPPORTED, "2D operators are not sharded (replicas only)");
  FDIGA_CHECK(!matrix_free || d == 3, FDIGA_ERR_NOT_SUPPORTED, "the matrix-free operator is 3D only");
  const bool ok_geo = geometry_id == FDIGA_GEOM_IDENTITY || (geometry_id == FDIGA_GEOM_ANNULUS && d == 2) ||
                      ((geometry_id == FDIGA_GEOM_DEFORMED_CUBE || geometry_id == FDIGA_GEOM_THICK_RING) && d == 3);
  FDIGA_CHECK(ok_geo, FDIGA_ERR_INVALID_ARG, "geometry %d not available in %dD", geometry_id, d);
  *out = nullptr;
  FDIGA_TRY(bind(ctx));
  Table1D T[3];
  int64_t n[3] = {1, 1, 1};
  for (int l = 0; l < d; ++l) {
    FDIGA_CHECK(ne[l] >= 1 && ne[l] + p - 2 >= 1, FDIGA_ERR_INVALID_ARG, "bad ne[%d]", l);
    build_table(p, ne[l], T[l]);
    n[l] = T[l].n;
  }
  fdiga_stencil* S = new_stencil(ctx, d, n);
  for (int l = 0; l < d; ++l) {
    S->hstart[l] = T[l].start;
    S->hwidth[l] = T[l].width;
  }
  int s = finish_stencil(S);
  std::vector<void*> tmp;
  auto dev_copy = [&](const void* h, size_t bytes, void** dptr) -> int {
    FDIGA_CUDA(cudaMalloc(dptr, bytes));
    tmp.push_back(*dptr);
    FDIGA_CUDA(cudaMemcpy(*dptr, h, bytes, cudaMemcpyHostToDevice));
    return FDIGA_OK;
  };
  AsmArgs A{};
  if (s == FDIGA_OK) {
    A.wmax = p + 1;
    A.n1 = n[0];
    A.n2 = n[1];
    A.n3 = n[2];
    A.S1 = S->hpre[0][n[0]];
    A.S2 = S->hpre[1][n[1]];
    A.geo.id = geometry_id;
    for (int k = 0; k < 4; ++k) A.geo.prm[k] = 0;
    const int np = geometry_id == FDIGA_GEOM_ANNULUS ? 2 : geometry_id == FDIGA_GEOM_DEFORMED_CUBE ? 1
                                                         : geometry_id == FDIGA_GEOM_THICK_RING  ? 3 : 0;
    FDIGA_CHECK(np == 0 || geo_params, FDIGA_ERR_INVALID_ARG, "geometry %d needs %d parameters", geometry_id, np);
    for (int k = 0; k < np; ++k) A.geo.prm[k] = geo_params[k];
    A.geo.wind = wind_id;
    for (int k = 0; k < 3; ++k) A.geo.wprm[k] = 0.0;
    FDIGA_CHECK(wind_id >= FDIGA_WIND_NONE && wind_id <= FDIGA_WIND_ROTATING, FDIGA_ERR_INVALID_ARG, "wind id %d",
                wind_id);
    const int nw = wind_id == FDIGA_WIND_CONSTANT ? d : wind_id == FDIGA_WIND_ROTATING ? 1 : 0;
    FDIGA_CHECK(nw == 0 || wind_params, FDIGA_ERR_INVALID_ARG, "wind %d needs %d parameters", wind_id, nw);
    for (int k = 0; k < nw; ++k) A.geo.wprm[k] = wind_params[k];
    const double* taus[3] = {nullptr, nullptr, nullptr};
    const double* tabs[3] = {nullptr, nullptr, nullptr};
    for (int l = 0; l < d && s == FDIGA_OK; ++l) {
      std::vector<double> tab;
      for (int r = 0; r < 3; ++r) tab.insert(tab.end(), T[l].val[r].begin(), T[l].val[r].end());
      void* dp = nullptr;
      s = dev_copy(T[l].tau.data(), n[l] * 8, &dp);
      taus[l] = (const double*)dp;
      if (s == FDIGA_OK) s = dev_copy(tab.data(), tab.size() * 8, &dp);
      tabs[l] = (const double*)dp;
    }
    A.tau1 = taus[0];
    A.tau2 = taus[1];
    A.tau3 = taus[2];
    A.tab1 = tabs[0];
    A.tab2 = tabs[1];
    A.tab3 = tabs[2];
    A.w1 = S->width[0];
    A.w2 = S->width[1];
    A.w3 = S->width[2];
    A.pre1 = S->pre[0];
    A.pre2 = S->pre[1];
    A.pre3 = S->pre[2];
    A.voff1 = S->voff1;
    A.wm1 = S->wm1;
  }
  if (s == FDIGA_OK && matrix_free) {
    // keep the 1D tables and the map; the 8^3 tiles' x boxes bound the shared memory of the kernel
    S->mf = true;
    S->mf_W = p + 1;
    S->mf_geo = A.geo;
    for (int l = 0; l < 3; ++l) {
      S->mf_tau[l] = const_cast<double*>(l == 0 ? A.tau1 : l == 1 ? A.tau2 : A.tau3);
      S->mf_tab[l] = const_cast<double*>(l == 0 ? A.tab1 : l == 1 ? A.tab2 : A.tab3);
      tmp.erase(std::remove(tmp.begin(), tmp.end(), (void*)S->mf_tau[l]), tmp.end());
      tmp.erase(std::remove(tmp.begin(), tmp.end(), (void*)S->mf_tab[l]), tmp.end());
      const int64_t first = (l == 2) ? S->o : 0, last = (l == 2) ? S->e : n[l];
      int bmax = 1;
      std::vector<int32_t> box;
      for (int64_t a0 = first; a0 < last; a0 += MF_T) {
        int hi0 = 0;
        for (int64_t i = a0; i < std::min<int64_t>(a0 + MF_T, last); ++i) {
          hi0 = std::max(hi0, S->hstart[l][i] + S->hwidth[l][i]);
          if (i > a0 && S->hstart[l][i] < S->hstart[l][i - 1]) s = FDIGA_ERR_NOT_SUPPORTED;
        }
        bmax = std::max(bmax, hi0 - S->hstart[l][a0]);
        box.push_back(S->hstart[l][a0]);
        box.push_back(hi0 - S->hstart[l][a0]);
      }
      S->mf_B[l] = bmax;
      if (box.empty()) box.assign(2, 0);
      if (cudaMalloc(&S->mf_box[l], box.size() * 4) != cudaSuccess ||
          cudaMemcpy(S->mf_box[l], box.data(), box.size() * 4, cudaMemcpyHostToDevice) != cudaSuccess)
        s = FDIGA_ERR_CUDA;
      // trigonometric factors of the map at the Greville points (setup, host libm)
      std::vector<double> trig(2 * n[l]);
      const double th = geo_theta(geometry_id);
      for (int64_t i = 0; i < n[l]; ++i) {
        trig[2 * i] = std::sin(th * T[l].tau[i]);
        trig[2 * i + 1] = std::cos(th * T[l].tau[i]);
      }
      if (cudaMalloc(&S->mf_trig[l], trig.size() * 8) != cudaSuccess ||
          cudaMemcpy(S->mf_trig[l], trig.data(), trig.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess)
        s = FDIGA_ERR_CUDA;
    }
    if (s == FDIGA_OK && matfree_smem_bytes(S->mf_B[0], S->mf_B[1], S->mf_B[2]) > 200 * 1024) {
      set_error("matrix-free operator: tile box %dx%dx%d exceeds shared memory", S->mf_B[0], S->mf_B[1], S->mf_B[2]);
      s = FDIGA_ERR_NOT_SUPPORTED;
    }
  }
  if (s == FDIGA_OK && !matrix_free) {
    cudaError_t e = cudaMalloc(&S->vals, (S->nnz + 2) * sizeof(double));
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    if (e == cudaSuccess) e = cudaMemsetAsync(S->vals, 0, (S->nnz + 2) * sizeof(double), ctx->stream);
    if (e == cudaSuccess) {
      A.vals = S->vals;
      A.row0 = S->o * n[0] * n[1];
      A.nrows = S->Nloc;
      A.vbase = S->vbase;
      const int64_t blocks = std::max<int64_t>(1, (S->Nloc + 127) / 128);
      if (d == 3)
        assemble_kernel<3><<<(unsigned)blocks, 128, 0, ctx->stream>>>(A);
      else
        assemble_kernel<2><<<(unsigned)blocks, 128, 0, ctx->stream>>>(A);
      count_launch(ctx);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(ctx->stream);
    if (e != cudaSuccess) {
      set_error("colloc_assemble: %s", cudaGetErrorString(e));
      s = FDIGA_ERR_CUDA;
    }
  }
  for (void* q : tmp) cudaFree(q);
  if (s != FDIGA_OK) {
    stencil_destroy(S);
    return s;
  }
  *out = S;
  return FDIGA_OK;
}

int colloc_assemble(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                    fdiga_stencil** out) {
  return colloc_build(ctx, d, p, ne, geometry_id, geo_params, FDIGA_WIND_NONE, nullptr, 0, out);
}

int colloc_matrix_free(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                       fdiga_stencil** out) {
  return colloc_build(ctx, d, p, ne, geometry_id, geo_params, FDIGA_WIND_NONE, nullptr, 1, out);
}

int colloc_assemble_cd(fdiga_ctx* ctx, int d, int p, const int64_t* ne, int geometry_id, const double* geo_params,
                       int wind_id, const double* wind_params, int matrix_free, fdiga_stencil** out) {
  return colloc_build(ctx, d, p, ne, geometry_id, geo_params, wind_id, wind_params, matrix_free ? 1 : 0, out);
}

int colloc_1d_convection(int p, int64_t ne, const double* wt, double* H) {
  FDIGA_CHECK(H && wt && p >= 1 && ne >= 1 && ne + p - 2 >= 1, FDIGA_ERR_INVALID_ARG,
              "bad colloc_1d_convection arguments");
  Table1D T;
  build_table(p, ne, T);
  const int64_t n = T.n;
  std::memset(H, 0, n * n * sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int c = 0; c < T.width[i]; ++c) H[i * n + T.start[i] + c] = wt[i] * T.val[1][i * T.wmax + c];
  return FDIGA_OK;
}

int stencil_matvec(fdiga_stencil* S, const double* x, double* y) {
  fdiga::NvtxRange nvtx_("fdiga:stencil_matvec");
  return fdiga::stencil_matvec_ex(S, x, y, nullptr);
}

}  // extern "C"

namespace fdiga {
int stencil_matvec_ex(fdiga_stencil* S, const double* x, double* y, const int* skip) {
  FDIGA_CHECK(S && ((x && y) || S->Nloc == 0), FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_CHECK(x != y || S->Nloc == 0, FDIGA_ERR_INVALID_ARG, "stencil_matvec: x and y must not alias");
  fdiga_ctx* ctx = S->ctx;
  FDIGA_TRY(bind(ctx));
  const bool sh = ctx->sharded;
  if (sh) {  // halo planes from the neighbouring slabs (collective: every rank takes part)
    std::vector<P2PMsg> snd = S->hsend;
    for (size_t i = 0; i < snd.size(); ++i)
      snd[i].ptr = const_cast<double*>(x) + (S->hsend_plane[i] - S->o) * S->n[0] * S->n[1];
    FDIGA_TRY(comm_exchange(ctx, snd, S->hrecv));
  }
  if (S->Nloc == 0) return FDIGA_OK;
  if (S->mf) {  // matrix-free sum-factorised operator (matfree.cu)
    MfArgs M{};
    M.n1 = S->n[0];
    M.n2 = S->n[1];
    M.n3 = S->n[2];
    M.o = S->o;
    M.e = S->e;
    M.lo = S->lo;
    M.t1 = (S->n[0] + MF_T - 1) / MF_T;
    M.t2 = (S->n[1] + MF_T - 1) / MF_T;
    M.t3 = (S->e - S->o + MF_T - 1) / MF_T;
    M.x = x;
    const int64_t plane = S->n[0] * S->n[1];
    M.halo_lo = S->halo;
    M.halo_hi = S->halo ? S->halo + (S->o - S->lo) * plane : nullptr;
    M.y = y;
    M.st1 = S->start[0];
    M.st2 = S->start[1];
    M.st3 = S->start[2];
    M.w1 = S->width[0];
    M.w2 = S->width[1];
    M.w3 = S->width[2];
    M.tab1 = S->mf_tab[0];
    M.tab2 = S->mf_tab[1];
    M.tab3 = S->mf_tab[2];
    M.tau1 = S->mf_tau[0];
    M.tau2 = S->mf_tau[1];
    M.tau3 = S->mf_tau[2];
    M.trig1 = S->mf_trig[0];
    M.trig2 = S->mf_trig[1];
    M.trig3 = S->mf_trig[2];
    M.box1 = S->mf_box[0];
    M.box2 = S->mf_box[1];
    M.box3 = S->mf_box[2];
    M.W = S->mf_W;
    M.B1 = S->mf_B[0];
    M.B2 = S->mf_B[1];
    M.B3 = S->mf_B[2];
    M.geo = S->mf_geo;
    M.skip = skip;
    M.sharded = sh ? 1 : 0;
    FDIGA_TRY(matfree_launch(M, ctx->stream));
    count_launch(ctx);
    return FDIGA_OK;
  }
  MvArgs A = make_mv_args(S, x, y);
  A.skip = skip;
  const unsigned grid = (unsigned)((S->Nloc + 255) / 256);
  // variant: batch UB window pairs per load phase; selectable for experiments with FDIGA_MV_VARIANT
  static int variant = -1;
  if (variant < 0) {
    const char* v = getenv("FDIGA_MV_VARIANT");
    variant = v ? atoi(v) : 1;
  }
  switch (S->wm1 * 10 + variant) {
#define FDIGA_MV_LAUNCH(W, UB, MB)                                                                      \
  if (sh)                                                                                              \
    matvec_kernel<W, UB, MB, true><<<grid, 256, 0, ctx->stream>>>(A);                                  \
  else                                                                                                 \
    matvec_kernel<W, UB, MB, false><<<grid, 256, 0, ctx->stream>>>(A);
#define FDIGA_MV_CASE(W)                                                     \
  case W * 10 + 0:                                                          \
    FDIGA_MV_LAUNCH(W, 1, 4)                                                \
    break;                                                                  \
  case W * 10 + 1:                                                          \
    FDIGA_MV_LAUNCH(W, 2, 3)                                                \
    break;                                                                  \
  case W * 10 + 2:                                                          \
    FDIGA_MV_LAUNCH(W, 3, 2)                                                \
    break;                                                                  \
  case W * 10 + 3:                                                          \
    FDIGA_MV_LAUNCH(W, 4, 2)                                                \
    break;
    FDIGA_MV_CASE(1)
    FDIGA_MV_CASE(2)
    FDIGA_MV_CASE(3)
    FDIGA_MV_CASE(4)
    FDIGA_MV_CASE(5)
    FDIGA_MV_CASE(6)
    FDIGA_MV_CASE(7)
    FDIGA_MV_CASE(8)
    FDIGA_MV_CASE(9)
    FDIGA_MV_CASE(10)
    FDIGA_MV_CASE(11)
#undef FDIGA_MV_CASE
#undef FDIGA_MV_LAUNCH
    default:
      FDIGA_CHECK(false, FDIGA_ERR_NOT_SUPPORTED, "window width %d / variant %d", S->wm1, variant);
  }
  count_launch(ctx);
  FDIGA_CUDA(cudaGetLastError());
  return FDIGA_OK;
}

int64_t stencil_local_rows(const fdiga_stencil* S) { return S->Nloc; }

}  // namespace fdiga

extern "C" {

int stencil_info(const fdiga_stencil* S, int64_t* nnz, int64_t* n_out, int32_t* start_l0, int32_t* width_l0) {
  FDIGA_CHECK(S, FDIGA_ERR_INVALID_ARG, "NULL stencil");
  if (nnz) *nnz = S->nnz;
  if (n_out)
    for (int l = 0; l < S->d; ++l) n_out[l] = S->n[l];
  if (start_l0) std::memcpy(start_l0, S->hstart[0].data(), S->n[0] * sizeof(int32_t));
  if (width_l0) std::memcpy(width_l0, S->hwidth[0].data(), S->n[0] * sizeof(int32_t));
  return FDIGA_OK;
}

int stencil_get_values(const fdiga_stencil* S, double* values_host) {
  FDIGA_CHECK(S && values_host, FDIGA_ERR_INVALID_ARG, "NULL argument");
  FDIGA_CHECK(!S->mf, FDIGA_ERR_NOT_SUPPORTED, "a matrix-free operator stores no values");
  FDIGA_TRY(bind(S->ctx));
  double* canon = nullptr;
  FDIGA_CUDA(cudaMalloc(&canon, S->nnz * sizeof(double)));
  int s = permute_values(const_cast<fdiga_stencil*>(S), S->vals, canon, 0);
  if (s == FDIGA_OK) {
    cudaError_t e = cudaMemcpy(values_host, canon, S->nnz * sizeof(double), cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) {
      set_error("stencil_get_values: %s", cudaGetErrorString(e));
      s = FDIGA_ERR_CUDA;
    }
  }
  cudaFree(canon);
  return s;
}

int colloc_1d_windows(int p, int64_t ne, int32_t* start, int32_t* width) {
  FDIGA_CHECK(start && width && p >= 1 && ne >= 1 && ne + p - 2 >= 1, FDIGA_ERR_INVALID_ARG,
              "bad colloc_1d_windows arguments");
  Table1D T;
  build_table(p, ne, T);
  std::memcpy(start, T.start.data(), T.n * sizeof(int32_t));
  std::memcpy(width, T.width.data(), T.n * sizeof(int32_t));
  return FDIGA_OK;
}

int colloc_1d_factors(int p, int64_t ne, double* M, double* K) {
  FDIGA_CHECK(M && K && p >= 1 && ne >= 1, FDIGA_ERR_INVALID_ARG, "bad colloc_1d_factors arguments");
  Table1D T;
  build_table(p, ne, T);
  const int64_t n = T.n;
  std::memset(M, 0, n * n * sizeof(double));
  std::memset(K, 0, n * n * sizeof(double));
  for (int64_t i = 0; i < n; ++i)
    for (int c = 0; c < T.width[i]; ++c) {
      M[i * n + T.start[i] + c] = T.val[0][i * T.wmax + c];
      K[i * n + T.start[i] + c] = -T.val[2][i * T.wmax + c];
    }
  return FDIGA_OK;
}

}  // extern "C"

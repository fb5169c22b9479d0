// Closed-form Jacobians / Hessians of the analytic geometry maps of the configs, shared by the
// assembly kernel (stencil.cu) and the matrix-free operator (matfree.cu).
#pragma once
#include "common.cuh"

namespace fdiga {

struct Geo {
  int id;
  double prm[4];
  int wind;      // FDIGA_WIND_*: convection-diffusion L_w = -Lap + w . grad (eq:convection); 0 = Poisson
  double wprm[3];
};

struct JH {
  double J[3][3];     // J[c][a] = dF_c / dxi_a
  double H[3][3][3];  // H[c][a][b] = d^2 F_c / dxi_a dxi_b
};

// Angular frequency of the trigonometric factors of a map: sin/cos(theta x_l) enter J and H.
__host__ __device__ __forceinline__ double geo_theta(int id) {
  return id == FDIGA_GEOM_DEFORMED_CUBE ? 3.141592653589793 : 0.5 * 3.141592653589793;
}

// Closed-form Jacobian and Hessians of the analytic maps (FDIGA_GEOM_*); unused entries are zero.
// sn[l], cs[l] = sin / cos(theta x_l) (geo_theta), evaluated by the caller (on the fly or from tables).
__device__ __forceinline__ JH geometry_jh(const Geo g, const double x0, const double sn[3], const double cs[3]) {
  JH r;
#pragma unroll
  for (int c = 0; c < 3; ++c)
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      r.J[c][a] = (c == a) ? 1.0 : 0.0;
#pragma unroll
      for (int b = 0; b < 3; ++b) r.H[c][a][b] = 0.0;
    }
  if (g.id == FDIGA_GEOM_ANNULUS || g.id == FDIGA_GEOM_THICK_RING) {
    const double r0 = g.prm[0], r1 = g.prm[1];
    const double dr = r1 - r0, w = geo_theta(g.id);
    const double rad = r0 + dr * x0;
    const double s1 = sn[1], c1 = cs[1];  // angle w xi_2
    r.J[0][0] = dr * c1;
    r.J[0][1] = -rad * w * s1;
    r.J[1][0] = dr * s1;
    r.J[1][1] = rad * w * c1;
    r.H[0][0][1] = -dr * w * s1;
    r.H[0][1][0] = -dr * w * s1;
    r.H[0][1][1] = -rad * w * w * c1;
    r.H[1][0][1] = dr * w * c1;
    r.H[1][1][0] = dr * w * c1;
    r.H[1][1][1] = -rad * w * w * s1;
    if (g.id == FDIGA_GEOM_THICK_RING) r.J[2][2] = g.prm[2];
  } else if (g.id == FDIGA_GEOM_DEFORMED_CUBE) {
    const double PI = geo_theta(g.id);
    const double amp = g.prm[0];
    const double s0 = sn[0], c0 = cs[0], s1 = sn[1], c1 = cs[1], s2 = sn[2], c2 = cs[2];
    const double gr[3] = {PI * c0 * s1 * s2, PI * s0 * c1 * s2, PI * s0 * s1 * c2};
    const double P2 = PI * PI;
    const double hd = -P2 * s0 * s1 * s2, h01 = P2 * c0 * c1 * s2, h02 = P2 * c0 * s1 * c2, h12 = P2 * s0 * c1 * c2;
    const double hg[3][3] = {{hd, h01, h02}, {h01, hd, h12}, {h02, h12, hd}};
#pragma unroll
    for (int c = 0; c < 3; ++c)
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        r.J[c][a] += amp * gr[a];
#pragma unroll
        for (int b = 0; b < 3; ++b) r.H[c][a][b] = amp * hg[a][b];
      }
  }
  return r;
}

// The map F(xi) itself (same trigonometric factors as geometry_jh).
__device__ __forceinline__ void geometry_F(const Geo g, const double x0, const double x1, const double x2,
                                           const double sn[3], const double cs[3], double F[3]) {
  F[0] = x0;
  F[1] = x1;
  F[2] = x2;
  if (g.id == FDIGA_GEOM_ANNULUS || g.id == FDIGA_GEOM_THICK_RING) {
    const double rad = g.prm[0] + (g.prm[1] - g.prm[0]) * x0;
    F[0] = rad * cs[1];
    F[1] = rad * sn[1];
    F[2] = g.id == FDIGA_GEOM_THICK_RING ? g.prm[2] * x2 : 0.0;
  } else if (g.id == FDIGA_GEOM_DEFORMED_CUBE) {
    const double bump = g.prm[0] * sn[0] * sn[1] * sn[2];
    F[0] += bump;
    F[1] += bump;
    F[2] += bump;
  }
}

// Physical wind w(x) (FDIGA_WIND_*): constant (wprm), or the rigid rotation omega (-x_2, x_1, 0).
__device__ __forceinline__ void wind_at(const Geo g, const double F[3], double w[3]) {
  w[0] = w[1] = w[2] = 0.0;
  if (g.wind == FDIGA_WIND_CONSTANT) {
    w[0] = g.wprm[0];
    w[1] = g.wprm[1];
    w[2] = g.wprm[2];
  } else if (g.wind == FDIGA_WIND_ROTATING) {
    w[0] = -g.wprm[0] * F[1];
    w[1] = g.wprm[0] * F[0];
  }
}

// Same, evaluating the trigonometric factors here.
__device__ __forceinline__ JH geometry_jh(const Geo g, const double x0, const double x1, const double x2) {
  const double th = geo_theta(g.id);
  double sn[3], cs[3];
  sincos(th * x0, &sn[0], &cs[0]);
  sincos(th * x1, &sn[1], &cs[1]);
  sincos(th * x2, &sn[2], &cs[2]);
  return geometry_jh(g, x0, sn, cs);
}

// Inverse of the leading D x D block by cofactors (one reciprocal of the determinant).
template <int D>
__device__ __forceinline__ void inv_small(const double A[3][3], double B[3][3]) {
  if (D == 2) {
    const double id = 1.0 / (A[0][0] * A[1][1] - A[0][1] * A[1][0]);
    B[0][0] = A[1][1] * id;
    B[0][1] = -A[0][1] * id;
    B[1][0] = -A[1][0] * id;
    B[1][1] = A[0][0] * id;
    return;
  }
  const double c00 = A[1][1] * A[2][2] - A[1][2] * A[2][1];
  const double c01 = A[1][2] * A[2][0] - A[1][0] * A[2][2];
  const double c02 = A[1][0] * A[2][1] - A[1][1] * A[2][0];
  const double id = 1.0 / (A[0][0] * c00 + A[0][1] * c01 + A[0][2] * c02);
  B[0][0] = c00 * id;
  B[1][0] = c01 * id;
  B[2][0] = c02 * id;
  B[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) * id;
  B[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) * id;
  B[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) * id;
  B[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) * id;
  B[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) * id;
  B[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) * id;
}

// Collocation coefficients at one point (eq:collocation, chain rule):
//   -Lap_x u = - sum_ab G_ab d_a d_b u^ + sum_a beta_a d_a u^,  G = (J^T J)^{-1},
//   beta_a = sum_c (J^{-1})_{ac} tr(G H_c).
// wphys (may be nullptr): the physical wind at the point; adds (J^{-1} w)_a to beta_a (w . grad_x u =
// (J^{-1} w) . grad_xi u^, NEXT-4).
template <int D>
__device__ __forceinline__ void colloc_coeffs(const JH& jh, double G[3][3], double beta[3],
                                              const double* wphys = nullptr) {
  double Ji[3][3];
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) Ji[a][b] = 0;
  inv_small<D>(jh.J, Ji);
  // G = (J^T J)^{-1} = J^{-1} J^{-T}
#pragma unroll
  for (int a = 0; a < 3; ++a)
#pragma unroll
    for (int b = 0; b < 3; ++b) {
      double s = 0;
#pragma unroll
      for (int c = 0; c < D; ++c) s += Ji[a][c] * Ji[b][c];
      G[a][b] = s;
    }
#pragma unroll
  for (int a = 0; a < 3; ++a) beta[a] = 0;
#pragma unroll
  for (int c = 0; c < D; ++c) {
    double tr = 0;  // tr(G H_c)
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int b = 0; b < D; ++b) tr += G[a][b] * jh.H[c][b][a];
#pragma unroll
    for (int a = 0; a < D; ++a) beta[a] += Ji[a][c] * tr;
  }
  if (wphys) {
#pragma unroll
    for (int a = 0; a < D; ++a)
#pragma unroll
      for (int c = 0; c < D; ++c) beta[a] += Ji[a][c] * wphys[c];
  }
}

}  // namespace fdiga

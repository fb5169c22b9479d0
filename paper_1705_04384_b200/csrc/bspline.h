// Host B-spline evaluation shared by the collocation tables (stencil.cu) and the weighted-quadrature
// rule (wq.cu): Piegl & Tiller's DersBasisFuns on open uniform knot vectors.
#pragma once
#include <algorithm>
#include <cstdint>
#include <vector>

namespace fdiga {

// Piegl & Tiller "DersBasisFuns": nonzero basis functions of degree p on the knot span `span`
// and their derivatives up to order nd, ders[k][r] for functions span-p+r, r = 0..p.
inline void ders_basis_funs(int span, double u, int p, int nd, const std::vector<double>& U,
                     std::vector<std::vector<double>>& ders) {
  std::vector<std::vector<double>> ndu(p + 1, std::vector<double>(p + 1));
  std::vector<double> left(p + 1), right(p + 1);
  ndu[0][0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = u - U[span + 1 - j];
    right[j] = U[span + j] - u;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      ndu[j][r] = right[r + 1] + left[j - r];
      double temp = ndu[r][j - 1] / ndu[j][r];
      ndu[r][j] = saved + right[r + 1] * temp;
      saved = left[j - r] * temp;
    }
    ndu[j][j] = saved;
  }
  ders.assign(nd + 1, std::vector<double>(p + 1, 0.0));
  for (int j = 0; j <= p; ++j) ders[0][j] = ndu[j][p];
  std::vector<std::vector<double>> a(2, std::vector<double>(p + 1));
  for (int r = 0; r <= p; ++r) {
    int s1 = 0, s2 = 1;
    a[0][0] = 1.0;
    for (int k = 1; k <= nd; ++k) {
      double dd = 0.0;
      int rk = r - k, pk = p - k;
      if (r >= k) {
        a[s2][0] = a[s1][0] / ndu[pk + 1][rk];
        dd = a[s2][0] * ndu[rk][pk];
      }
      int j1 = (rk >= -1) ? 1 : -rk;
      int j2 = (r - 1 <= pk) ? k - 1 : p - r;
      for (int j = j1; j <= j2; ++j) {
        a[s2][j] = (a[s1][j] - a[s1][j - 1]) / ndu[pk + 1][rk + j];
        dd += a[s2][j] * ndu[rk + j][pk];
      }
      if (r <= pk) {
        a[s2][k] = -a[s1][k - 1] / ndu[pk + 1][r];
        dd += a[s2][k] * ndu[r][pk];
      }
      ders[k][r] = dd;
      std::swap(s1, s2);
    }
  }
  int r = p;
  for (int k = 1; k <= nd; ++k) {
    for (int j = 0; j <= p; ++j) ders[k][j] *= r;
    r *= (p - k);
  }
}


// Open uniform knot vector with ne elements and degree p: {0}^{p+1}, k / ne, {1}^{p+1}.
inline std::vector<double> open_knots(int p, int64_t ne) {
  std::vector<double> U;
  for (int k = 0; k <= p; ++k) U.push_back(0.0);
  for (int64_t k = 1; k < ne; ++k) U.push_back((double)k / (double)ne);
  for (int k = 0; k <= p; ++k) U.push_back(1.0);
  return U;
}

// Values of the derivative of order `deriv` (<= 2) of ALL interior functions j = 1..n at x (full index
// j -> out[j - 1]); half-open spans, left limit at x = 1.
inline void interior_values(int p, int64_t ne, const std::vector<double>& U, double x, int deriv, double* out) {
  const int64_t m = ne + p, n = m - 2;
  for (int64_t j = 0; j < n; ++j) out[j] = 0.0;
  int span = p;
  while (span < m - 1 && U[span + 1] <= x) ++span;
  std::vector<std::vector<double>> ders;
  ders_basis_funs(span, x, p, std::min(deriv, p), U, ders);
  for (int r = 0; r <= p; ++r) {
    const int64_t k = span - p + r;  // full index
    if (k >= 1 && k <= n) out[k - 1] = deriv <= p ? ders[deriv][r] : 0.0;
  }
}

}  // namespace fdiga

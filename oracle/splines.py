"""Univariate B-spline spaces (oracle; test infrastructure only).

P:144-148  open knot vector Xi = {xi_1..xi_{m+p+1}}, basis B_0..B_{m-1} of degree p.
P:157-159  interior functions i = 1..m-2 (Dirichlet functions B_0, B_{m-1} removed), n = m-2.
P:163-164  Greville abscissae tau_i = (1/p) sum_{j=1}^p xi_{i+j+1} (1-based xi), i = 1..n.
P:180      (M^C)_{ij} = B_j(tau_i),  (K^C)_{ij} = -B''_j(tau_i).

The basis is evaluated by the textbook Cox-de Boor recursion written out over ALL
m functions (no local-support shortcuts), with the left-limit convention at x = 1
(SPEC.md:91).
"""
import numpy as np


def open_uniform_knots(ne: int, p: int) -> np.ndarray:
    """Open knot vector with ne uniform elements, interior knots of multiplicity 1.

    xi = {0}^{p+1} U {k/ne}_{k=1}^{ne-1} U {1}^{p+1};  length m+p+1 with m = ne+p.
    """
    if ne < 1 or p < 1:
        raise ValueError("need ne >= 1 and p >= 1")
    interior = [k / ne for k in range(1, ne)]
    return np.array([0.0] * (p + 1) + interior + [1.0] * (p + 1), dtype=np.float64)


def _degree0(knots: np.ndarray, x: float) -> np.ndarray:
    """B_{k,0}(x) = 1 on [xi_k, xi_{k+1}), 0 elsewhere; at x = 1 the last non-empty span is closed."""
    nk = len(knots)
    B = np.zeros(nk - 1)
    for k in range(nk - 1):
        if knots[k] <= x < knots[k + 1]:
            B[k] = 1.0
    if x >= knots[-1]:
        # left limit at the right end: the last non-degenerate span owns x = 1
        for k in range(nk - 2, -1, -1):
            if knots[k] < knots[k + 1]:
                B[k] = 1.0
                break
    return B


def basis_all(knots: np.ndarray, p: int, x: float, deriv: int = 0) -> np.ndarray:
    """Values of B^{(deriv)}_k(x), k = 0..m-1, for all m = len(knots)-p-1 functions of degree p.

    Cox-de Boor:  B_{k,q} = (x-xi_k)/(xi_{k+q}-xi_k) B_{k,q-1} + (xi_{k+q+1}-x)/(xi_{k+q+1}-xi_{k+1}) B_{k+1,q-1}
    Derivative:   d/dx B_{k,q} = q/(xi_{k+q}-xi_k) B_{k,q-1} - q/(xi_{k+q+1}-xi_{k+1}) B_{k+1,q-1}
    (terms with a zero denominator are 0).  The derivative rule is applied `deriv` times,
    i.e. B^{(r)}_{k,q} = q [ B^{(r-1)}_{k,q-1}/(xi_{k+q}-xi_k) - B^{(r-1)}_{k+1,q-1}/(xi_{k+q+1}-xi_{k+1}) ].
    """
    if not (0.0 <= x <= 1.0):
        raise ValueError("x outside [0,1]")

    def rec(q: int, r: int) -> np.ndarray:
        # array over k = 0..len(knots)-q-2 of B^{(r)}_{k,q}(x)
        if q == 0:
            B0 = _degree0(knots, x)
            return B0 if r == 0 else np.zeros_like(B0)
        nfun = len(knots) - q - 1
        out = np.zeros(nfun)
        if r == 0:
            low = rec(q - 1, 0)
            for k in range(nfun):
                d1 = knots[k + q] - knots[k]
                d2 = knots[k + q + 1] - knots[k + 1]
                a = (x - knots[k]) / d1 * low[k] if d1 > 0 else 0.0
                b = (knots[k + q + 1] - x) / d2 * low[k + 1] if d2 > 0 else 0.0
                out[k] = a + b
        else:
            low = rec(q - 1, r - 1)
            for k in range(nfun):
                d1 = knots[k + q] - knots[k]
                d2 = knots[k + q + 1] - knots[k + 1]
                a = low[k] / d1 if d1 > 0 else 0.0
                b = low[k + 1] / d2 if d2 > 0 else 0.0
                out[k] = q * (a - b)
        return out

    return rec(p, deriv)


def greville_interior(knots: np.ndarray, p: int) -> np.ndarray:
    """tau_i = (1/p) sum_{j=1}^p xi_{i+j+1}, i = 1..n (1-based xi)."""
    m = len(knots) - p - 1
    n = m - 2
    xi1 = np.concatenate([[np.nan], knots])   # 1-based view
    return np.array([sum(xi1[i + j + 1] for j in range(1, p + 1)) / p for i in range(1, n + 1)])


def greville_full(knots: np.ndarray, p: int) -> np.ndarray:
    """Greville points of the full basis k = 0..m-1: (1/p) sum_{j=1}^p xi_{k+j} (0-based xi).  Used by pins."""
    m = len(knots) - p - 1
    return np.array([knots[k + 1:k + p + 1].sum() / p for k in range(m)])


def colloc_1d(ne: int, p: int):
    """1D collocation factors at the interior Greville points.

    Returns (tau, M, K, D1) with, for i, j = 1..n (0-based rows/cols here),
      M[i,j]  = B_j(tau_i),  K[i,j] = -B''_j(tau_i),  D1[i,j] = B'_j(tau_i)
    where B_j is interior function j (full index j, j = 1..m-2).
    """
    knots = open_uniform_knots(ne, p)
    tau = greville_interior(knots, p)
    n = len(tau)
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    D1 = np.zeros((n, n))
    for i, t in enumerate(tau):
        M[i] = basis_all(knots, p, t, 0)[1:n + 1]
        D1[i] = basis_all(knots, p, t, 1)[1:n + 1]
        K[i] = -basis_all(knots, p, t, 2)[1:n + 1]
    return tau, M, K, D1


def colloc_1d_convection(ne: int, p: int, wt):
    """1D convection factor of the collocation analogue of eq:convec_prec_2:
    H[i, j] = w~(tau_i) B'_j(tau_i) at the interior Greville points (wt: scalar or the n values w~(tau_i)).
    The collocation counterpart of the paper's Galerkin H_l = int w~ B_i B'_j (reading 17)."""
    tau, M, K, D1 = colloc_1d(ne, p)
    wt = np.broadcast_to(np.asarray(wt, dtype=np.float64), tau.shape)
    return wt[:, None] * D1


def flatten_index(mi, n: int) -> int:
    """1-based multi-index (i_1..i_d) -> scalar i = 1 + sum_l n^{l-1}(i_l - 1)."""
    return 1 + sum((n ** l) * (il - 1) for l, il in enumerate(mi))


def galerkin_1d(ne: int, p: int, wind: float = 0.0):
    """Univariate Galerkin factors on the interior functions (eq:univariateG P:357):

      M_ij = int_0^1 B_i B_j,   K_ij = int_0^1 B'_i B'_j,   H_ij = int_0^1 w B_i B'_j  (constant wind w),

    by Gauss-Legendre quadrature with p+1 points per element (exact: the integrands are polynomials of
    degree <= 2p on every element).  Used for the convection-diffusion preconditioner eq:convec_prec_2
    (P:363), whose pencils (K + H, M) have complex eigenvalue pairs for strong wind.
    """
    knots = open_uniform_knots(ne, p)
    m = len(knots) - p - 1
    n = m - 2
    gx, gw = np.polynomial.legendre.leggauss(p + 1)
    M = np.zeros((n, n))
    K = np.zeros((n, n))
    H = np.zeros((n, n))
    breaks = np.unique(knots)
    for e in range(len(breaks) - 1):
        a, b = breaks[e], breaks[e + 1]
        for xq, wq in zip(gx, gw):
            x = 0.5 * (a + b) + 0.5 * (b - a) * xq
            w = 0.5 * (b - a) * wq
            B = basis_all(knots, p, x, 0)[1:n + 1]
            D = basis_all(knots, p, x, 1)[1:n + 1]
            M += w * np.outer(B, B)
            K += w * np.outer(D, D)
            H += w * wind * np.outer(B, D)
    return M, K, H

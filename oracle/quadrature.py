"""Gauss rules, weighted quadrature (WQ) and the WQ-Galerkin operator (oracle; test infrastructure only).

P:186-193: Galerkin stiffness (A_G)_ij = sum_{alpha,beta} int c_{alpha beta}(xi) d_alpha B^_i d_beta B^_j dxi with
           c = Q(xi) = det(J) J^{-1} K J^{-T} (eq:Q), K = I.
P:195-199: weighted quadrature (eq:WQapprox): (A_wq)_ij = sum_{alpha,beta} sum_q c_{alpha beta}(x_q) w^{alpha beta}_{iq}
           d_beta B^_j(x_q), the test function folded into the weights, exact when c is constant
           (Calabro et al. 2017).  A_wq is in general nonsymmetric.
P:204-214: on the identity map A_wq = A_G = the Kronecker forms eq:wq2D / eq:wq3D with the exact 1D Galerkin
           factors (eq:univariateWQ).
Readings (reading 18, SPEC.md quadrature module): quadrature points = all knot-span endpoints and
midpoints; for row i and derivative pair (a, b) the weights live on the points of supp(B_i) and satisfy
sum_q w^{ab}_{iq} B_j^{(b)}(x_q) = int B_i^{(a)} B_j^{(b)} for every interior j overlapping i (minimum-norm
solution of the underdetermined moment system).  Multivariate weights are tensor products:
w^{alpha beta}_{i q} = prod_l w_l^{(a_l b_l)}_{i_l q_l} with a_l = [l = alpha], b_l = [l = beta].
"""
import numpy as np
import scipy.sparse as sp

from . import geometry as geo
from .splines import basis_all, open_uniform_knots


def gauss_rule(ne: int, p: int, q: int = None):
    """Gauss-Legendre with q (default p + 1) points on every element of [0,1] split uniformly into ne."""
    q = q or p + 1
    gx, gw = np.polynomial.legendre.leggauss(q)
    xs, ws = [], []
    for e in range(ne):
        a, b = e / ne, (e + 1) / ne
        xs.append(0.5 * (a + b) + 0.5 * (b - a) * gx)
        ws.append(0.5 * (b - a) * gw)
    return np.concatenate(xs), np.concatenate(ws)


def interior_values(ne: int, p: int, x, deriv: int):
    """E[q, j] = B_j^{(deriv)}(x_q) for the interior functions j = 1..n (full index j)."""
    knots = open_uniform_knots(ne, p)
    n = ne + p - 2
    return np.array([basis_all(knots, p, float(t), deriv)[1:n + 1] for t in x])


def wq_points(ne: int, p: int):
    """Knot-span endpoints and midpoints of the uniform partition (2 ne + 1 points, the rule's base set), plus
    the quarter points of the first and last p elements; those are used only by rows whose moment system
    is rank-deficient on the base set (even p near the open-knot boundary; reading 18)."""
    pts = set(np.arange(2 * ne + 1) / (2 * ne))
    for k in list(range(min(p, ne))) + list(range(max(0, ne - p), ne)):
        pts.update([(k + 0.25) / ne, (k + 0.75) / ne])
    return np.array(sorted(pts))


def wq_rule_1d(ne: int, p: int):
    """Returns (xq, W, E): W[(a, b)] is the n x nq weight matrix of rows i, E[b] the nq x n matrix B_j^{(b)}(x_q)."""
    knots = open_uniform_knots(ne, p)
    n = ne + p - 2
    xq = wq_points(ne, p)
    E = {b: interior_values(ne, p, xq, b) for b in (0, 1)}
    xg, wg = gauss_rule(ne, p, p + 2)
    G = {b: interior_values(ne, p, xg, b) for b in (0, 1)}
    W = {}
    for a in (0, 1):
        for b in (0, 1):
            Wab = np.zeros((n, len(xq)))
            for i in range(n):
                lo, hi = knots[i + 1], knots[i + p + 2]              # supp(B_i), full index i + 1
                insupp = (xq >= lo - 1e-14) & (xq <= hi + 1e-14)
                base = np.abs(xq * 2 * ne - np.round(xq * 2 * ne)) < 1e-9   # endpoints and midpoints
                js = [j for j in range(n) if abs(i - j) <= p]       # interior trial functions overlapping row i
                mom = np.array([np.sum(wg * G[a][:, i] * G[b][:, j]) for j in js])
                for qs in (np.nonzero(insupp & base)[0], np.nonzero(insupp)[0]):
                    Bm = E[b][np.ix_(qs, js)].T                      # (#j) x (#q)
                    # minimum-norm solution (the system is consistent but rank-deficient for b = 1: the
                    # derivatives of the 2p + 1 functions living on supp(B_i) sum to zero there)
                    w, *_ = np.linalg.lstsq(Bm, mom, rcond=None)
                    if np.linalg.norm(Bm @ w - mom) <= 1e-11 * max(1.0, np.linalg.norm(mom)):
                        break
                else:
                    raise ValueError("WQ moment system not solvable")
                Wab[i, qs] = w
            W[(a, b)] = Wab
    return xq, W, E


def _kron(mats):
    """(x)_{l=d..1} mats[l] (mats given for l = 1..d)."""
    out = sp.csr_matrix(mats[0])
    for m in mats[1:]:
        out = sp.kron(sp.csr_matrix(m), out, format="csr")
    return out


def _grid(x, d):
    """Tensor grid of 1D points, flattened with the first coordinate fastest: (P, d)."""
    g = np.meshgrid(*([x] * d), indexing="ij")
    return np.stack([gi.transpose(tuple(range(d - 1, -1, -1))).reshape(-1) for gi in g], axis=1)


def q_matrix(geometry: int, xi, params=()):
    """Q(xi) = det(J) J^{-1} J^{-T} (eq:Q with K = I) and det(J) at the points xi (P, d)."""
    _, J, _ = geo.evaluate(geometry, xi, params)
    Jinv = np.linalg.inv(J)
    det = np.linalg.det(J)
    return det[:, None, None] * np.einsum("pac,pbc->pab", Jinv, Jinv), det


class WQDiscretisation:
    """WQ-Galerkin operator A_wq (eq:WQapprox) and the exact Galerkin A_G (Gauss) on an analytic map."""

    def __init__(self, d, p, ne, geometry, params=()):
        self.d, self.p, self.ne, self.geometry, self.params = d, p, ne, geometry, tuple(params)
        self.n = ne + p - 2
        self.N = self.n ** d
        self.xq, self.W, self.E = wq_rule_1d(ne, p)

    def assemble_wq(self):
        d = self.d
        Q, _ = q_matrix(self.geometry, _grid(self.xq, d), self.params)
        A = None
        for al in range(d):
            for be in range(d):
                Wk = _kron([self.W[(int(l == al), int(l == be))] for l in range(d)])
                Ek = _kron([self.E[int(l == be)] for l in range(d)])
                term = Wk @ sp.diags(Q[:, al, be]) @ Ek
                A = term if A is None else A + term
        return A.tocsr()

    def _gauss_forms(self):
        d, p, ne = self.d, self.p, self.ne
        xg, wg = gauss_rule(ne, p, p + 2)
        G = {b: interior_values(ne, p, xg, b) for b in (0, 1)}
        pts = _grid(xg, d)
        wt = _grid(wg, d).prod(axis=1)
        Q, det = q_matrix(self.geometry, pts, self.params)
        return G, wt, Q, det

    def assemble_galerkin(self):
        """A_G by Gauss quadrature (p + 2 points per element): the exact Galerkin stiffness of P:188."""
        d = self.d
        G, wt, Q, _ = self._gauss_forms()
        A = None
        for al in range(d):
            for be in range(d):
                Gi = _kron([G[int(l == al)] for l in range(d)])
                Gj = _kron([G[int(l == be)] for l in range(d)])
                term = Gi.T @ sp.diags(wt * Q[:, al, be]) @ Gj
                A = term if A is None else A + term
        return A.tocsr()

    def h1_gram(self):
        """H^1(Omega) Gram matrix of the interior basis: mass + stiffness in physical space (Table 1's H)."""
        d = self.d
        G, wt, Q, det = self._gauss_forms()
        G0 = _kron([G[0]] * d)
        M = G0.T @ sp.diags(wt * np.abs(det)) @ G0
        return (M + self.assemble_galerkin()).tocsr()

    def matvec(self, x):
        return self.assemble_wq() @ x


def e_h(disc: WQDiscretisation):
    """e_h = || H^{-1/2} (A_wq - A_G) H^{-1/2} ||_2 (Table 1), dense (small sizes only)."""
    E = (disc.assemble_wq() - disc.assemble_galerkin()).toarray()
    L = np.linalg.cholesky(disc.h1_gram().toarray())
    X = np.linalg.solve(L, np.linalg.solve(L, E.T).T)
    return float(np.linalg.norm(X, 2))

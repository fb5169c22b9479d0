"""Collocation operator A_C on an analytic geometry (oracle; test infrastructure only).

P:165-171 (eq:collocation, eq:collocationsystem): row i of A_C is the collocation condition at
F(tau_i), i.e.  (A_C)_{ij} = (L (B_j o F^{-1}))(F(tau_i)),  L u = -div(K grad u) with K = I.

Chain rule (written out in DESIGN.md "Readings", derivation for x = F(xi), u(x) = u^(xi)):
    Hess_xi u^ = J^T (Hess_x u) J + sum_c (grad_x u)_c H_c
    => -Lap_x u = - sum_{a,b} G_ab d_a d_b u^  +  sum_a beta_a d_a u^,
    G = (J^T J)^{-1},   beta_a = sum_c (J^{-1})_{ac} tr(G H_c).
With d_a d_b B^_j(tau_i) = prod_l D_l^{(t_l)}[i_l, j_l], t = e_a + e_b (tensor-product basis),
D^{(0)} = M^C, D^{(1)} = B', D^{(2)} = B'' = -K^C, the operator is
    A_C = sum_{a,b} diag(-G_ab) (x)_l D_l^{(e_a+e_b)_l}  +  sum_a diag(beta_a) (x)_l D_l^{(e_a)_l}
with (x)_l ordered D_d (x) ... (x) D_1 (i_1 fastest).
For the identity map G = I, beta = 0 and this is exactly eq:colloc2D / eq:colloc3D.

Convection-diffusion (NEXT-4; eq:convection P:345, L_w = -Lap + w . grad): grad_x u = J^{-T} grad_xi u^, so
w . grad_x u = (J^{-1} w) . grad_xi u^ and the first-order coefficient becomes beta_a + (J^{-1} w(F(tau)))_a.
"""
import numpy as np
import scipy.sparse as sp

from . import geometry as geo
from .splines import colloc_1d


class Discretisation:
    """1D factors + pointwise geometry coefficients for one (d, p, ne, geometry)."""

    def __init__(self, d, p, ne, geometry, params=(), wind=0, wind_params=()):
        self.d, self.p, self.ne, self.geometry, self.params = d, p, ne, geometry, tuple(params)
        self.wind, self.wind_params = wind, tuple(wind_params)
        tau, M, K, D1 = colloc_1d(ne, p)
        self.tau, self.M, self.K, self.D1 = tau, M, K, D1
        self.n = len(tau)
        self.N = self.n ** d
        # D^{(0)}, D^{(1)}, D^{(2)} (same 1D space in every direction)
        self.D = [M, D1, -K]
        self._coeffs = None

    # -- collocation points in flattened order (i_1 fastest) --
    def points(self):
        n, d = self.n, self.d
        grids = np.meshgrid(*([self.tau] * d), indexing="ij")   # grids[k][i_1..i_d] = tau[i_{k+1}]
        # C-order flattening of an array indexed [i_d, ..., i_1] has i_1 fastest
        return np.stack([g.transpose(tuple(range(d - 1, -1, -1))).reshape(-1) for g in grids], axis=1)

    def coefficients(self):
        """G (N, d, d) and beta (N, d) at every collocation point F(tau_i)."""
        if self._coeffs is None:
            xi = self.points()
            F, J, H = geo.evaluate(self.geometry, xi, self.params)
            Jinv = np.linalg.inv(J)
            G = np.linalg.inv(np.einsum("pca,pcb->pab", J, J))            # (J^T J)^{-1}
            trGH = np.einsum("pab,pcba->pc", G, H)                         # tr(G H_c) for each c
            beta = np.einsum("pac,pc->pa", Jinv, trGH)
            if self.wind:
                beta = beta + np.einsum("pac,pc->pa", Jinv, geo.wind(self.wind, F, self.wind_params))
            self._coeffs = (G, beta)
        return self._coeffs

    def terms(self):
        """List of (coefficient vector c_t (N,), derivative orders t = (t_1..t_d))."""
        G, beta = self.coefficients()
        d = self.d
        out = []
        for a in range(d):
            for b in range(d):
                t = [0] * d
                t[a] += 1
                t[b] += 1
                out.append((-G[:, a, b], tuple(t)))
        for a in range(d):
            t = [0] * d
            t[a] = 1
            out.append((beta[:, a], tuple(t)))
        return out

    # -- operators --
    def kron_factor(self, t):
        """Sparse D_d^{(t_d)} (x) ... (x) D_1^{(t_1)}."""
        mats = [sp.csr_matrix(self.D[t[l]]) for l in range(self.d)]
        out = mats[0]
        for l in range(1, self.d):
            out = sp.kron(mats[l], out, format="csr")
        return out

    def assemble_csr(self):
        """A_C as a scipy CSR matrix (small configurations only)."""
        A = None
        for c, t in self.terms():
            term = sp.diags(c) @ self.kron_factor(t)
            A = term if A is None else A + term
        A = A.tocsr()
        A.eliminate_zeros()
        return A

    def matvec(self, x):
        """y = A_C x by the sum-factorised form: sum_t c_t * ((x)_l D_l^{(t_l)}) x (mode products)."""
        X = x.reshape((self.n,) * self.d)          # X[i_d, ..., i_1]
        y = np.zeros(self.N)
        for c, t in self.terms():
            Y = X
            for l in range(self.d):
                axis = self.d - 1 - l                  # direction l+1 acts on axis d-1-l
                Y = np.moveaxis(np.tensordot(self.D[t[l]], Y, axes=([1], [axis])), 0, axis)
            y += c * Y.reshape(-1)
        return y

    def row(self, i_flat):
        """Explicit row i of A_C: dict {j_flat: value} over the 1D supports, from the chain-rule formula."""
        n, d = self.n, self.d
        idx = [(i_flat // n ** l) % n for l in range(d)]     # (i_1..i_d), 0-based
        vals = {}
        for c, t in self.terms():
            cols = [np.nonzero(self.D[t[l]][idx[l]])[0] for l in range(d)]
            for jj in np.array(np.meshgrid(*cols, indexing="ij")).reshape(d, -1).T:
                v = c[i_flat]
                for l in range(d):
                    v *= self.D[t[l]][idx[l], jj[l]]
                j = int(sum(jj[l] * n ** l for l in range(d)))
                vals[j] = vals.get(j, 0.0) + v
        return vals


def kron_preconditioner_dense(Ms, Ks):
    """Dense P = sum_k ( (x)_{l=d..1} (K_l if l == k else M_l) )  (eq:colloc2D/3D)."""
    d = len(Ms)
    P = 0
    for k in range(d):
        mats = [Ks[l] if l == k else Ms[l] for l in range(d)]
        T = mats[0]
        for l in range(1, d):
            T = np.kron(mats[l], T)
        P = P + T
    return P


def kron_preconditioner_sparse(Ms, Ks):
    d = len(Ms)
    P = None
    for k in range(d):
        mats = [sp.csr_matrix(Ks[l] if l == k else Ms[l]) for l in range(d)]
        T = mats[0]
        for l in range(1, d):
            T = sp.kron(mats[l], T, format="csr")
        P = T if P is None else P + T
    return P.tocsr()

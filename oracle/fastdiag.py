"""Fast-Diagonalization (FD) preconditioner, nonsymmetric version (oracle; test infrastructure only).

P:418-422 (eq:eigendecomposition)  M_l^{-1} K_l U_l = U_l D_l.
P:424      V_l := (M_l U_l)^{-T};  M_l = V_l^{-T} U_l^{-1},  K_l = V_l^{-T} D_l U_l^{-1}.
P:430      (eq:FD2D) s = (U_2 (x) U_1)(D_2 (x) I + I (x) D_1)^{-1}(V_2 (x) V_1)^T b.
P:444      (eq:FD3D) s = (U_3 (x) U_2 (x) U_1)(D_3(x)I(x)I + I(x)D_2(x)I + I(x)I(x)D_1)^{-1}(V_3(x)V_2(x)V_1)^T b.
P:448-450  Remark 1: real spectrum, diagonalizable with well-conditioned U (assumed; guarded here).

Conventions (readings 1-5): W_l := V_l^T = (M_l U_l)^{-1} is the forward factor;
columns of U_l have unit 2-norm and eigenvalues are sorted ascending;
|Im lambda| <= 1e-8 rho and cond(U) <= 1e8 are the guards.
"""
import numpy as np
import scipy.linalg as sla


class FDFactors:
    """Per-direction (U_l, W_l, lam_l), l = 1..d (list index l-1)."""

    def __init__(self, U, W, lam):
        self.U = [np.asarray(u, dtype=np.float64) for u in U]
        self.W = [np.asarray(w, dtype=np.float64) for w in W]
        self.lam = [np.asarray(v, dtype=np.float64) for v in lam]
        self.d = len(self.U)
        self.n = [u.shape[0] for u in self.U]


def setup_direction(M, K, tol_imag=1e-8, cond_max=1e8):
    """Generalized eigendecomposition of the pencil (K, M): K U = M U D (eq:eigendecomposition).

    Returns (U, W, lam) with W = (M U)^{-1} (= V^T).  Raises on a complex spectrum or
    an ill-conditioned U (Remark 1).
    """
    w, U = sla.eig(K, M)
    rho = np.max(np.abs(w))
    if np.max(np.abs(w.imag)) > tol_imag * rho:
        raise ValueError("complex spectrum (Remark 1 violated)")
    lam = w.real
    U = U.real
    order = np.argsort(lam, kind="stable")
    lam, U = lam[order], U[:, order]
    U = U / np.linalg.norm(U, axis=0)
    if np.linalg.cond(U) > cond_max:
        raise ValueError("ill-conditioned eigenvector matrix")
    W = np.linalg.inv(M @ U)
    return U, W, lam


def setup(Ms, Ks, **kw):
    out = [setup_direction(M, K, **kw) for M, K in zip(Ms, Ks)]
    return FDFactors([o[0] for o in out], [o[1] for o in out], [o[2] for o in out])


def factors_from_eig(U, lam, M=None):
    """Factors from a given eigenbasis: W = (M U)^{-1}, M = I if omitted (cfg4: W = U^{-1})."""
    W = [np.linalg.inv(u if M is None else M[l] @ u) for l, u in enumerate(U)]
    return FDFactors(U, W, lam)


def lambda_sum(f: FDFactors):
    """Lambda[i] = sum_l lam_l[i_l] in flattened order (i_1 fastest): the diagonal of sum_l I(x)..D_l..(x)I."""
    d = f.d
    L = np.zeros([f.n[l] for l in range(d - 1, -1, -1)])
    for l in range(d):
        shape = [1] * d
        shape[d - 1 - l] = f.n[l]
        L = L + f.lam[l].reshape(shape)
    return L.reshape(-1)


def mode_apply(mats, x, ns):
    """((x)_{l=d..1} A_l) x by mode products: A_l acts on index i_l (axis d-l of X[i_d..i_1])."""
    d = len(mats)
    X = x.reshape([ns[l] for l in range(d - 1, -1, -1)])
    for l in range(d):
        axis = d - 1 - l
        X = np.moveaxis(np.tensordot(mats[l], X, axes=([1], [axis])), 0, axis)
    return X.reshape(-1)


def apply(f: FDFactors, b):
    """s = P^{-1} b by eq:FD2D / eq:FD3D, step by step:
       1. b~ = (W_d (x) ... (x) W_1) b        (the (V_d (x) ... (x) V_1)^T product)
       2. s~ = b~ / Lambda                    ("just a diagonal scaling")
       3. s  = (U_d (x) ... (x) U_1) s~
    """
    bt = mode_apply(f.W, b, f.n)
    st = bt / lambda_sum(f)
    return mode_apply(f.U, st, f.n)


def apply_loops(f: FDFactors, b):
    """Same as apply(), written as explicit per-entry sums (tiny n only; brute-force pin)."""
    d, ns = f.d, f.n
    N = int(np.prod(ns))
    idx = [np.unravel_index(i, ns[::-1])[::-1] for i in range(N)]   # (i_1..i_d) for flat i
    bt = np.zeros(N)
    for i in range(N):
        acc = 0.0
        for j in range(N):
            w = 1.0
            for l in range(d):
                w *= f.W[l][idx[i][l], idx[j][l]]
            acc += w * b[j]
        bt[i] = acc
    st = np.array([bt[i] / sum(f.lam[l][idx[i][l]] for l in range(d)) for i in range(N)])
    s = np.zeros(N)
    for i in range(N):
        acc = 0.0
        for j in range(N):
            u = 1.0
            for l in range(d):
                u *= f.U[l][idx[i][l], idx[j][l]]
            acc += u * st[j]
        s[i] = acc
    return s


def flops(ns):
    """Algorithmic flops of one apply: 2 passes x d mode products x 2 N n_l  (= 12 n^4 in 3D; 8 n^3 in 2D)."""
    N = int(np.prod(ns))
    return 4 * N * int(sum(ns))

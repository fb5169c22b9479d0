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
    """Per-direction (U_l, W_l, lam_l[, lam_im_l]), l = 1..d (list index l-1).

    Real 2x2 blocks: a complex pair a +- ib with eigenvector p + iq occupies two adjacent
    columns (p, q) of U_l; lam[j] = lam[j+1] = a and lam_im[j] = +b, lam_im[j+1] = -b, and the
    corresponding block of D_l is [[a, b], [-b, a]] (M^{-1}K [p q] = [p q] [[a, b], [-b, a]]).
    """

    def __init__(self, U, W, lam, lam_im=None):
        self.U = [np.asarray(u, dtype=np.float64) for u in U]
        self.W = [np.asarray(w, dtype=np.float64) for w in W]
        self.lam = [np.asarray(v, dtype=np.float64) for v in lam]
        self.d = len(self.U)
        self.n = [u.shape[0] for u in self.U]
        self.lam_im = ([np.zeros(n) for n in self.n] if lam_im is None
                       else [np.asarray(v, dtype=np.float64) for v in lam_im])

    @property
    def has_pairs(self):
        return any(np.any(v != 0) for v in self.lam_im)

    def D(self, l):
        """The (block-)diagonal D_l of eq:eigendecomposition / P:434 as a dense matrix."""
        n = self.n[l]
        D = np.diag(self.lam[l]).astype(np.float64)
        j = 0
        while j < n:
            if self.lam_im[l][j] != 0:
                D[j, j + 1] = self.lam_im[l][j]
                D[j + 1, j] = self.lam_im[l][j + 1]
                j += 2
            else:
                j += 1
        return D


def setup_direction(M, K, tol_imag=1e-8, cond_max=1e8, allow_complex=False):
    """Generalized eigendecomposition of the pencil (K, M): K U = M U D (eq:eigendecomposition).

    Returns (U, W, lam, lam_im) with W = (M U)^{-1} (= V^T).  Complex pairs are kept in real
    2x2-block form when allow_complex, else rejected; an ill-conditioned U is rejected
    (Remark 1).  Order: ascending real part, pairs adjacent (+b column first).
    """
    w, Uc = sla.eig(K, M)
    rho = np.max(np.abs(w))
    is_c = np.abs(w.imag) > tol_imag * rho
    if np.any(is_c) and not allow_complex:
        raise ValueError("complex spectrum (Remark 1 violated)")
    cols, lam, lam_im = [], [], []
    # one representative per pair: the member with positive imaginary part
    keys = [j for j in range(len(w)) if not is_c[j] or w[j].imag > 0]
    keys.sort(key=lambda j: (w[j].real, 0 if not is_c[j] else 1))
    for j in keys:
        if not is_c[j]:
            u = Uc[:, j].real
            cols.append(u / np.linalg.norm(u))
            lam.append(w[j].real)
            lam_im.append(0.0)
        else:
            p, q = Uc[:, j].real, Uc[:, j].imag   # eigenvalue a + ib, eigenvector p + iq
            s = np.sqrt((p @ p + q @ q) / 2)
            cols += [p / s, q / s]
            lam += [w[j].real, w[j].real]
            lam_im += [w[j].imag, -w[j].imag]
    U = np.array(cols).T
    if np.linalg.cond(U) > cond_max:
        raise ValueError("ill-conditioned eigenvector matrix")
    W = np.linalg.inv(M @ U)
    return U, W, np.array(lam), np.array(lam_im)


def setup(Ms, Ks, **kw):
    out = [setup_direction(M, K, **kw) for M, K in zip(Ms, Ks)]
    return FDFactors([o[0] for o in out], [o[1] for o in out], [o[2] for o in out], [o[3] for o in out])


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


def _groups(f: FDFactors, l):
    """Index groups of D_l: (j,) for a real eigenvalue, (j, j+1) for a complex pair."""
    out, j = [], 0
    while j < f.n[l]:
        if f.lam_im[l][j] != 0:
            out.append((j, j + 1))
            j += 2
        else:
            out.append((j,))
            j += 1
    return out


def block_solve(f: FDFactors, bt):
    """s~ = Lambda^{-1} b~ with Lambda = sum_l I (x)..(x) D_l (x)..(x) I block diagonal: one small
    dense solve per product of index groups (blocks of size 1, 2, 4 or 8)."""
    import itertools
    d, ns = f.d, f.n
    st = np.empty_like(bt)
    Ds = [f.D(l) for l in range(d)]
    for combo in itertools.product(*[_groups(f, l) for l in range(d - 1, -1, -1)]):
        gs = combo[::-1]                                     # gs[l] = group of direction l
        blk = 0
        for l in range(d):
            T = None
            for m in range(d - 1, -1, -1):                  # kron order d..1 (i_1 fastest)
                f_m = Ds[m][np.ix_(gs[m], gs[m])] if m == l else np.eye(len(gs[m]))
                T = f_m if T is None else np.kron(T, f_m)
            blk = blk + T
        flat = []
        for jj in itertools.product(*[gs[m] for m in range(d - 1, -1, -1)]):   # C order over (j_d..j_1)
            j = jj[::-1]
            idx, stride = 0, 1
            for m in range(d):
                idx += j[m] * stride
                stride *= ns[m]
            flat.append(idx)
        st[flat] = np.linalg.solve(blk, bt[flat])
    return st


def apply(f: FDFactors, b):
    """s = P^{-1} b by eq:FD2D / eq:FD3D, step by step:
       1. b~ = (W_d (x) ... (x) W_1) b        (the (V_d (x) ... (x) V_1)^T product)
       2. s~ = b~ / Lambda                    ("just a diagonal scaling"; small block solves
                                               for complex pairs kept as real 2x2 blocks)
       3. s  = (U_d (x) ... (x) U_1) s~
    """
    bt = mode_apply(f.W, b, f.n)
    st = block_solve(f, bt) if f.has_pairs else bt / lambda_sum(f)
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

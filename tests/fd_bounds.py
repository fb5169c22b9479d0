"""Elementwise a-priori error bounds for the FD apply (test infrastructure, plain numpy; no oracle or
library arithmetic).  Used by the GPU accuracy tests (test_gpu_fp64_contract.py) and pinned on the CPU
(test_int8_split_scheme.py) against exact rational arithmetic.

The apply is a chain of mode products y = F x along one tensor axis (K = the contraction length) and one
pointwise divide by Lambda (eq:FD3D).  For an input known up to an elementwise error E (|x^ - x| <= E):

  IEEE FP64 dot products (DMMA path, and the numpy oracle):  the classical bound
      |y^ - y| <= |F| E + gamma_K |F| (|x| + E),          gamma_K = K u / (1 - K u),  u = 2^-53
  int8-split tensor-core product (the path's accuracy contract):
      |y^ - y| <= |F| E + 8 u |F| (|x| + E) + 2^-51.9 K max_k (|x_k| + E_k) max_k |F_ik|
    (the digits keep 55 bits of every fibre / factor row relative to its maximum; the dropped digit pairs and
    the FP64 combination of the integer accumulators add the rest), plus gamma_K |F|(|x| + E) for the outputs
    the guard recomputes as IEEE FP64 dot products (added everywhere: an upper bound of the max of the two)
  divide z = y / Lambda (Lambda > 0 here):  |z^ - z| <= E / Lambda + 2 u |z|

Vectors are (n3, n2, n1) arrays (i1 fastest); axis l = 0, 1, 2 is the mode-(l+1) contraction.
"""
import numpy as np

U = 2.0 ** -53


def gamma(K):
    return K * U / (1 - K * U)


def mode(F, x, l):
    """y = F x along tensor axis l (0: i1, the last array axis; 2: i3, the first)."""
    ax = 2 - l
    return np.moveaxis(np.tensordot(F, x, axes=([1], [ax])), 0, ax)


def fibre_max(x, l):
    return np.max(np.abs(x), axis=2 - l, keepdims=True)


def factor_row_max(F, l):
    """max_k |F_ik| broadcast along axis l of the output."""
    shape = [1, 1, 1]
    shape[2 - l] = F.shape[0]
    return np.max(np.abs(F), axis=1).reshape(shape)


def product_bound(F, x, E, l, path):
    """Error bound of y = F x (x exact up to E) on `path` ('fp64' or 'int8'), and y itself."""
    K = F.shape[1]
    y = mode(F, x, l)
    absF = np.abs(F)
    ax = np.abs(x) + E
    B = mode(absF, E, l) + gamma(K) * mode(absF, ax, l)
    if path == "int8":
        B = B + 8 * U * mode(absF, ax, l) + 2.0 ** -51.9 * K * fibre_max(ax, l) * factor_row_max(F, l)
    return y, B


def apply_bound(Ws, Us, lam_sum, x, path, bwd=(2, 1, 0)):
    """(s, B): s = (U3 (x) U2 (x) U1) Lambda^-1 (W3 (x) W2 (x) W1) x evaluated in FP64 and the elementwise
    bound of the error of `path` for it, propagated through the chain: forward modes 1, 2, 3, the divide,
    backward modes in the order `bwd` (the library: 3, 2, 1; the oracle's mode_apply: 1, 2, 3).
    lam_sum: Lambda as an (n3, n2, n1) array."""
    E = np.zeros_like(x)
    y = x
    for l in range(3):
        y, E = product_bound(Ws[l], y, E, l, path)
    z = y / lam_sum
    E = E / np.abs(lam_sum) + 2 * U * np.abs(z)
    y = z
    for l in bwd:
        y, E = product_bound(Us[l], y, E, l, path)
    return y, E


def lam_grid(lams):
    """Lambda[i3, i2, i1] = lam_1[i1] + lam_2[i2] + lam_3[i3]."""
    l1, l2, l3 = lams
    return l3[:, None, None] + l2[None, :, None] + l1[None, None, :]

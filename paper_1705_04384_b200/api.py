"""Thin Python binding over libfdiga.so (include/fdiga.h), same names as the C ABI.

Marshalling only: host matrices come in as numpy float64 arrays (copied by the library), device
vectors as torch float64 CUDA tensors (their data_ptr is passed through), and every step of the
hot path runs in the library's kernels.  torch provides device memory and streams only.
"""
import ctypes as C
import weakref

import numpy as np

from ._lib import (BicgstabOpts, BicgstabReport, FdSetupOpts, GmresOpts, GmresReport, c_double_p, c_int32_p, c_int64_p, check, load)

ORTH_CGS_DGKS = 0
ORTH_CGS2 = 1
ORTH_DCGS2 = 2


def _dptr(a):
    return a.ctypes.data_as(c_double_p)


def _host_f64(a, shape=None):
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if shape is not None and a.shape != tuple(shape):
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _devptr(t, n=None):
    import torch
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("expected a contiguous float64 CUDA tensor")
    if n is not None and t.numel() != n:
        raise ValueError(f"expected {n} elements, got {t.numel()}")
    return C.c_void_p(t.data_ptr())


def nccl_unique_id():
    """A fresh 128-byte ncclUniqueId (rank 0 creates it, every rank passes it to Context)."""
    buf = C.create_string_buffer(128)
    check(load().fdiga_nccl_unique_id(buf), "fdiga_nccl_unique_id")
    return buf.raw


def partition(n, nparts, part):
    """Balanced split of [0, n) into nparts ranges (fdiga_partition): the range [begin, end) of `part`."""
    b, e = C.c_int64(), C.c_int64()
    check(load().fdiga_partition(int(n), int(nparts), int(part), C.byref(b), C.byref(e)), "fdiga_partition")
    return b.value, e.value


def transpose_plan(n_inner, n_last, nranks, rank):
    """Exchange schedule of the sharded FD mode-d pass (fdiga_transpose_plan): four int64 arrays
    (slab_off, slab_cnt, tr_off, tr_cnt) of length nranks, in doubles."""
    arrs = [np.zeros(nranks, np.int64) for _ in range(4)]
    check(load().fdiga_transpose_plan(int(n_inner), int(n_last), int(nranks), int(rank),
                                      *[a.ctypes.data_as(c_int64_p) for a in arrs]), "fdiga_transpose_plan")
    return tuple(arrs)


def halo_plan(start, width, nranks, rank):
    """Halo schedule of the sharded matvec (fdiga_halo_plan): (lo, hi, send_b, send_e, recv_b, recv_e)."""
    st = np.ascontiguousarray(start, dtype=np.int32)
    wd = np.ascontiguousarray(width, dtype=np.int32)
    lo, hi = C.c_int64(), C.c_int64()
    arrs = [np.zeros(nranks, np.int64) for _ in range(4)]
    check(load().fdiga_halo_plan(st.size, st.ctypes.data_as(c_int32_p), wd.ctypes.data_as(c_int32_p), int(nranks),
                                 int(rank), C.byref(lo), C.byref(hi), *[a.ctypes.data_as(c_int64_p) for a in arrs]),
          "fdiga_halo_plan")
    return (lo.value, hi.value) + tuple(arrs)


def colloc_1d_windows(p, ne):
    """The 1D column windows (start, width) of the stored operator (host only)."""
    n = ne + p - 2
    st, wd = np.empty(n, np.int32), np.empty(n, np.int32)
    check(load().colloc_1d_windows(int(p), int(ne), st.ctypes.data_as(c_int32_p), wd.ctypes.data_as(c_int32_p)),
          "colloc_1d_windows")
    return st, wd


class LoopbackHub:
    """fdiga_loopback: nranks contexts in one process on one device (one host thread per rank)."""

    def __init__(self, nranks):
        self._lib = load()
        h = C.c_void_p()
        check(self._lib.fdiga_loopback_create(int(nranks), C.byref(h)), "fdiga_loopback_create")
        self.handle, self.nranks = h, nranks

    def close(self):
        if self.handle:
            check(self._lib.fdiga_loopback_destroy(self.handle), "fdiga_loopback_destroy")
            self.handle = None


class Context:
    """fdiga_ctx: a device, a stream and (optionally) a process group (NCCL, or a loopback hub)."""

    def __init__(self, device=0, stream=None, nranks=1, rank=0, nccl_unique_id=None, hub=None):
        lib = load()
        self._lib = lib
        h = C.c_void_p()
        s = C.c_void_p(stream) if stream is not None else None
        if hub is not None:
            check(lib.fdiga_ctx_create_loopback(int(device), s, hub.handle, int(rank), C.byref(h)),
                  "fdiga_ctx_create_loopback")
            nranks = hub.nranks
        else:
            uid = C.c_char_p(bytes(nccl_unique_id)) if nccl_unique_id is not None else None
            check(lib.fdiga_ctx_create(int(device), s, int(nranks), int(rank), uid, C.byref(h)), "fdiga_ctx_create")
        self.handle = h
        self.device = device
        self.nranks, self.rank = int(nranks), int(rank)
        self._children = weakref.WeakSet()  # plans / operators: destroyed before the context (C ABI rule)

    def slab(self, n_last):
        b, e = C.c_int64(), C.c_int64()
        check(self._lib.fdiga_slab(self.handle, int(n_last), C.byref(b), C.byref(e)), "fdiga_slab")
        return b.value, e.value

    def kernel_launches(self):
        return int(self._lib.fdiga_kernel_launches(self.handle))

    def close(self):
        if self.handle:
            for child in list(self._children):
                child.close()
            self._lib.fdiga_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class FDPlan:
    """fd_plan: per-direction factors (U_l, W_l = (M_l U_l)^{-1}, lam_l) resident on the device."""

    def __init__(self, ctx, handle, ns):
        self.ctx, self.handle, self.n = ctx, handle, list(ns)
        ctx._children.add(self)
        self.N_global = int(np.prod(self.n))
        self.slab = ctx.slab(self.n[-1])           # this rank's planes of the last axis
        self.N = (self.slab[1] - self.slab[0]) * (self.N_global // self.n[-1])   # local vector length

    def factors(self, l):
        n = self.n[l]
        U, W = np.empty((n, n)), np.empty((n, n))
        lr, li = np.empty(n), np.empty(n)
        check(self.ctx._lib.fd_get_factors(self.handle, l, _dptr(U), _dptr(W), _dptr(lr), _dptr(li)),
              "fd_get_factors")
        return U, W, lr, li

    def flops(self):
        return float(self.ctx._lib.fd_apply_flops(self.handle))

    def path(self):
        """('dmma' | 'int8_split', int8 tensor-core ops per apply) -- the kernel family of the mode products."""
        ops = C.c_double(0.0)
        k = self.ctx._lib.fd_plan_path(self.handle, C.byref(ops))
        if k < 0:
            check(k, "fd_plan_path")
        return ("int8_split" if k == 1 else "dmma"), float(ops.value)

    def set_path(self, path):
        """Select the mode-product kernels: 'dmma' (IEEE FP64) or 'int8_split' (fd_plan_set_path)."""
        code = {"dmma": 0, "int8_split": 1}[path]
        check(self.ctx._lib.fd_plan_set_path(self.handle, code), "fd_plan_set_path")

    def close(self):
        if self.handle:
            if self.ctx.handle:  # a closed context already destroyed its children
                self.ctx._lib.fd_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Stencil:
    """fdiga_stencil: the stored collocation operator A_C."""

    def __init__(self, ctx, handle):
        self.ctx, self.handle = ctx, handle
        ctx._children.add(self)
        nnz = C.c_int64()
        n = (C.c_int64 * 3)(1, 1, 1)
        check(ctx._lib.stencil_info(handle, C.byref(nnz), n, None, None), "stencil_info")
        self.nnz = nnz.value                       # values stored on this rank
        self.n = [n[0], n[1], n[2]]
        self.N_global = n[0] * n[1] * n[2]
        self.slab = ctx.slab(n[2]) if ctx.nranks > 1 else (0, n[2])
        self.N = (self.slab[1] - self.slab[0]) * n[0] * n[1]   # local rows

    def windows(self):
        """(start, width) of the column windows of direction 1 (int32 arrays of length n_1)."""
        st = np.empty(self.n[0], np.int32)
        wd = np.empty(self.n[0], np.int32)
        check(self.ctx._lib.stencil_info(self.handle, None, None, st.ctypes.data_as(c_int32_p),
                                         wd.ctypes.data_as(c_int32_p)), "stencil_info")
        return st, wd

    def values(self):
        out = np.empty(self.nnz)
        check(self.ctx._lib.stencil_get_values(self.handle, _dptr(out)), "stencil_get_values")
        return out

    def close(self):
        if self.handle:
            if self.ctx.handle:
                self.ctx._lib.stencil_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _mat_array(mats, ns):
    arrs = [_host_f64(m, (n, n)) for m, n in zip(mats, ns)]
    return arrs, (c_double_p * len(arrs))(*[_dptr(a) for a in arrs])


def _vec_array(vecs, ns):
    arrs = [_host_f64(v, (n,)) for v, n in zip(vecs, ns)]
    return arrs, (c_double_p * len(arrs))(*[_dptr(a) for a in arrs])


def fd_setup(ctx, M, K, tol_imag=1e-8, cond_max=1e8, allow_complex_pairs=False):
    d = len(M)
    ns = [np.asarray(m).shape[0] for m in M]
    n = (C.c_int64 * d)(*ns)
    am, pm = _mat_array(M, ns)
    ak, pk = _mat_array(K, ns)
    opts = FdSetupOpts(tol_imag, cond_max, int(allow_complex_pairs))
    h = C.c_void_p()
    check(ctx._lib.fd_setup(ctx.handle, d, n, pm, pk, C.byref(opts), C.byref(h)), "fd_setup")
    return FDPlan(ctx, h, ns)


def fd_setup_from_factors(ctx, U, W, lam):
    d = len(U)
    ns = [np.asarray(u).shape[0] for u in U]
    n = (C.c_int64 * d)(*ns)
    au, pu = _mat_array(U, ns)
    aw, pw = _mat_array(W, ns)
    al, pl = _vec_array(lam, ns)
    h = C.c_void_p()
    check(ctx._lib.fd_setup_from_factors(ctx.handle, d, n, pu, pw, pl, C.byref(h)), "fd_setup_from_factors")
    return FDPlan(ctx, h, ns)


def fd_setup_from_blocks(ctx, U, W, lam_re, lam_im):
    """Factors with complex pairs in real 2x2-block form; see include/fdiga.h."""
    d = len(U)
    ns = [np.asarray(u).shape[0] for u in U]
    n = (C.c_int64 * d)(*ns)
    au, pu = _mat_array(U, ns)
    aw, pw = _mat_array(W, ns)
    al, pl = _vec_array(lam_re, ns)
    ai, pi = _vec_array(lam_im, ns)
    h = C.c_void_p()
    check(ctx._lib.fd_setup_from_blocks(ctx.handle, d, n, pu, pw, pl, pi, C.byref(h)), "fd_setup_from_blocks")
    return FDPlan(ctx, h, ns)


def fd_setup_from_eig(ctx, U, lam, M=None):
    d = len(U)
    ns = [np.asarray(u).shape[0] for u in U]
    n = (C.c_int64 * d)(*ns)
    au, pu = _mat_array(U, ns)
    al, pl = _vec_array(lam, ns)
    pm = None
    if M is not None:
        amm, pm = _mat_array(M, ns)
    h = C.c_void_p()
    check(ctx._lib.fd_setup_from_eig(ctx.handle, d, n, pu, pl, pm, C.byref(h)), "fd_setup_from_eig")
    return FDPlan(ctx, h, ns)


def fd_apply(plan, r, s):
    """s = P^{-1} r on the device (asynchronous on the context stream)."""
    check(plan.ctx._lib.fd_apply(plan.handle, _devptr(r, plan.N), _devptr(s, plan.N)), "fd_apply")
    return s


def fd_apply_timed(plan, r, s):
    """One apply with per-kernel CUDA-event durations: list of (kind, ms), kind in {'dmma', 'split', 'int8_gemm',
    'slab_pack', 'exchange'} (collective on sharded plans)."""
    cap = 64
    ms = (C.c_float * cap)()
    kind = (C.c_int32 * cap)()
    cnt = C.c_int(0)
    check(plan.ctx._lib.fd_apply_timed(plan.handle, _devptr(r, plan.N), _devptr(s, plan.N), ms, kind, cap,
                                       C.byref(cnt)), "fd_apply_timed")
    names = {0: "dmma", 1: "split", 2: "int8_gemm", 3: "slab_pack", 4: "exchange"}
    return [(names[kind[k]], float(ms[k])) for k in range(min(cnt.value, cap))]


def fd_apply_host(plan, r_host, s_host):
    """Same with host (numpy, ideally pinned) buffers; H2D + apply + D2H inside the call."""
    if r_host.dtype != np.float64 or s_host.dtype != np.float64 or r_host.size != plan.N or s_host.size != plan.N:
        raise ValueError("fd_apply_host: float64 host arrays of the local length expected")
    check(plan.ctx._lib.fd_apply_host(plan.handle, _dptr(r_host), _dptr(s_host)), "fd_apply_host")
    return s_host


def fd_apply_host_async(plan, r_host, s_host):
    """Streaming host-buffer apply (double-buffered, overlapped copies); complete with fd_host_sync."""
    if r_host.dtype != np.float64 or s_host.dtype != np.float64 or r_host.size != plan.N or s_host.size != plan.N:
        raise ValueError("fd_apply_host_async: float64 host arrays of the local length expected")
    check(plan.ctx._lib.fd_apply_host_async(plan.handle, _dptr(r_host), _dptr(s_host)), "fd_apply_host_async")
    return s_host


def fd_host_sync(plan):
    check(plan.ctx._lib.fd_host_sync(plan.handle), "fd_host_sync")


def colloc_assemble(ctx, d, p, ne, geometry, geo_params=(), matrix_free=False, wind=0, wind_params=()):
    """The collocation operator A_C: stored tensor-window values (colloc_assemble) or, with
    matrix_free=True, the sum-factorised on-the-fly operator (colloc_matrix_free, 3D).  wind != 0: the
    convection-diffusion operator -Lap + w . grad (colloc_assemble_cd, NEXT-4)."""
    nes = [ne] * d if np.isscalar(ne) else list(ne)
    n = (C.c_int64 * d)(*nes)
    prm = np.ascontiguousarray(np.asarray(list(geo_params) + [0.0] * 4, dtype=np.float64))
    h = C.c_void_p()
    if wind:
        wp = np.ascontiguousarray(np.asarray(list(wind_params) + [0.0] * 3, dtype=np.float64))
        check(ctx._lib.colloc_assemble_cd(ctx.handle, d, int(p), n, int(geometry), _dptr(prm), int(wind), _dptr(wp),
                                          int(bool(matrix_free)), C.byref(h)), "colloc_assemble_cd")
        return Stencil(ctx, h)
    fn = ctx._lib.colloc_matrix_free if matrix_free else ctx._lib.colloc_assemble
    check(fn(ctx.handle, d, int(p), n, int(geometry), _dptr(prm), C.byref(h)),
          "colloc_matrix_free" if matrix_free else "colloc_assemble")
    return Stencil(ctx, h)


def stencil_create(ctx, n, start, width, values):
    d = len(n)
    nn = (C.c_int64 * d)(*n)
    st = [np.ascontiguousarray(np.asarray(s, dtype=np.int32)) for s in start]
    wd = [np.ascontiguousarray(np.asarray(w, dtype=np.int32)) for w in width]
    pst = (c_int32_p * d)(*[a.ctypes.data_as(c_int32_p) for a in st])
    pwd = (c_int32_p * d)(*[a.ctypes.data_as(c_int32_p) for a in wd])
    h = C.c_void_p()
    try:
        import torch
        on_dev = isinstance(values, torch.Tensor) and values.is_cuda
    except ImportError:
        on_dev = False
    if on_dev:
        vp = _devptr(values)
    else:
        values = _host_f64(values)
        vp = C.c_void_p(values.ctypes.data)
    check(ctx._lib.stencil_create(ctx.handle, d, nn, pst, pwd, vp, int(on_dev), C.byref(h)), "stencil_create")
    return Stencil(ctx, h)


def stencil_matvec(A, x, y):
    check(A.ctx._lib.stencil_matvec(A.handle, _devptr(x, A.N), _devptr(y, A.N)), "stencil_matvec")
    return y


def colloc_1d_convection(p, ne, wt):
    """H[i][j] = wt[i] B'_j(tau_i) (host), wt scalar or the n values of the univariate wind."""
    n = ne + p - 2
    w = np.ascontiguousarray(np.broadcast_to(np.asarray(wt, dtype=np.float64), (n,)))
    H = np.empty((n, n))
    check(load().colloc_1d_convection(int(p), int(ne), _dptr(w), _dptr(H)), "colloc_1d_convection")
    return H


def wq_assemble(ctx, d, p, ne, geometry, geo_params=()):
    """The weighted-quadrature Galerkin operator A_wq (NEXT-3) in the tensor-window layout."""
    prm = np.ascontiguousarray(np.asarray(list(geo_params) + [0.0] * 4, dtype=np.float64))
    h = C.c_void_p()
    check(ctx._lib.wq_assemble(ctx.handle, int(d), int(p), int(ne), int(geometry), _dptr(prm), C.byref(h)),
          "wq_assemble")
    return Stencil(ctx, h)


def galerkin_1d_factors(p, ne):
    """Univariate Galerkin factors M = int B_i B_j, K = int B'_i B'_j (host)."""
    n = ne + p - 2
    M, K = np.empty((n, n)), np.empty((n, n))
    check(load().galerkin_1d_factors(int(p), int(ne), _dptr(M), _dptr(K)), "galerkin_1d_factors")
    return M, K


def colloc_1d_factors(p, ne):
    n = ne + p - 2
    M, K = np.empty((n, n)), np.empty((n, n))
    check(load().colloc_1d_factors(int(p), int(ne), _dptr(M), _dptr(K)), "colloc_1d_factors")
    return M, K


def gmres_solve(ctx, A, P, b, x, m=30, rtol=1e-8, max_iters=1000, orth=ORTH_DCGS2, use_x0=False,
                history=False, raise_on_nonconvergence=True, profile=False):
    """Right-preconditioned GMRES(m); returns the report as a dict.  profile=True: eagerly launched cycles with
    the per-stage device times t_fd_ms / t_matvec_ms / t_orth_ms / t_comm_ms / t_other_ms (include/fdiga.h)."""
    opts = GmresOpts(int(m), float(rtol), int(max_iters), int(orth), int(use_x0), int(bool(profile)))
    rep = GmresReport()
    hist = None
    if history:
        hist = np.zeros(max_iters)
        rep.history = _dptr(hist)
        rep.history_cap = max_iters
    st = ctx._lib.gmres_solve(ctx.handle, A.handle, P.handle if P is not None else None, _devptr(b, A.N),
                              _devptr(x, A.N), C.byref(opts), C.byref(rep))
    if st != 0 and (raise_on_nonconvergence or st not in (-8, -9)):  # NOT_CONVERGED / BREAKDOWN reported
        check(st, "gmres_solve")
    out = dict(iters=rep.iters, restarts=rep.restarts, converged=bool(rep.converged), reorth=rep.reorth,
               rel_res_true=rep.rel_res_true, rel_res_implicit=rep.rel_res_implicit, t_total_ms=rep.t_total_ms,
               status=st)
    if profile:
        out.update(t_fd_ms=rep.t_fd_ms, t_matvec_ms=rep.t_matvec_ms, t_orth_ms=rep.t_orth_ms,
                   t_comm_ms=rep.t_comm_ms, t_other_ms=rep.t_other_ms)
    if hist is not None:
        out["history"] = hist[:rep.iters].copy()
    return out


def bicgstab_solve(ctx, A, P, b, x, rtol=1e-8, max_iters=1000, use_x0=False, history=False,
                   raise_on_failure=True):
    """Right-preconditioned BiCGStab (the paper's solver); returns the report as a dict (iters is a
    half-iteration count)."""
    opts = BicgstabOpts(float(rtol), int(max_iters), int(use_x0))
    rep = BicgstabReport()
    hist = None
    if history:
        hist = np.zeros(2 * max_iters)
        rep.history = _dptr(hist)
        rep.history_cap = 2 * max_iters
    st = ctx._lib.bicgstab_solve(ctx.handle, A.handle, P.handle if P is not None else None, _devptr(b, A.N),
                                 _devptr(x, A.N), C.byref(opts), C.byref(rep))
    if st != 0 and (raise_on_failure or st not in (-8, -9)):
        check(st, "bicgstab_solve")
    out = dict(iters=rep.iters, converged=bool(rep.converged), breakdown=bool(rep.breakdown), half=bool(rep.half),
               rel_res_true=rep.rel_res_true, rel_res_recursive=rep.rel_res_recursive, t_total_ms=rep.t_total_ms,
               status=st)
    if hist is not None:
        out["history"] = hist[:int(round(2 * rep.iters))].copy()
    return out

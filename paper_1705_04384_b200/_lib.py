"""ctypes declarations of the libfdiga.so C ABI (include/fdiga.h).  Argument marshalling only."""
import ctypes as C
import os

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FDIGA_LIB") or os.path.join(_PKG, "lib", "libfdiga.so")  # override: experiments

c_int64_p = C.POINTER(C.c_int64)
c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)


class FdSetupOpts(C.Structure):
    _fields_ = [("tol_imag", C.c_double), ("cond_max", C.c_double), ("allow_complex_pairs", C.c_int)]


class GmresOpts(C.Structure):
    _fields_ = [("m", C.c_int), ("rtol", C.c_double), ("max_iters", C.c_int), ("orth", C.c_int),
                ("use_x0", C.c_int), ("profile", C.c_int)]


class GmresReport(C.Structure):
    _fields_ = [("iters", C.c_int), ("restarts", C.c_int), ("converged", C.c_int), ("reorth", C.c_int),
                ("rel_res_true", C.c_double), ("rel_res_implicit", C.c_double), ("t_total_ms", C.c_double),
                ("history", c_double_p), ("history_cap", C.c_int),
                ("t_fd_ms", C.c_double), ("t_matvec_ms", C.c_double), ("t_orth_ms", C.c_double),
                ("t_comm_ms", C.c_double), ("t_other_ms", C.c_double)]


class BicgstabOpts(C.Structure):
    _fields_ = [("rtol", C.c_double), ("max_iters", C.c_int), ("use_x0", C.c_int)]


class BicgstabReport(C.Structure):
    _fields_ = [("iters", C.c_double), ("converged", C.c_int), ("breakdown", C.c_int), ("half", C.c_int),
                ("rel_res_true", C.c_double), ("rel_res_recursive", C.c_double), ("t_total_ms", C.c_double),
                ("history", c_double_p), ("history_cap", C.c_int)]


# name -> (restype, argtypes); every symbol include/fdiga.h declares
SIGNATURES = {
    "fdiga_ctx_create": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.POINTER(C.c_void_p)]),
    "fdiga_ctx_destroy": (C.c_int, [C.c_void_p]),
    "fdiga_slab": (C.c_int, [C.c_void_p, C.c_int64, c_int64_p, c_int64_p]),
    "fdiga_nccl_unique_id": (C.c_int, [C.c_void_p]),
    "fdiga_loopback_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
    "fdiga_loopback_destroy": (C.c_int, [C.c_void_p]),
    "fdiga_ctx_create_loopback": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "fdiga_partition": (C.c_int, [C.c_int64, C.c_int, C.c_int, c_int64_p, c_int64_p]),
    "fdiga_transpose_plan": (C.c_int, [C.c_int64, C.c_int64, C.c_int, C.c_int, c_int64_p, c_int64_p, c_int64_p,
                                       c_int64_p]),
    "fdiga_halo_plan": (C.c_int, [C.c_int64, c_int32_p, c_int32_p, C.c_int, C.c_int, c_int64_p, c_int64_p,
                                  c_int64_p, c_int64_p, c_int64_p, c_int64_p]),
    "colloc_1d_windows": (C.c_int, [C.c_int, C.c_int64, c_int32_p, c_int32_p]),
    "fdiga_status_string": (C.c_char_p, [C.c_int]),
    "fdiga_last_error": (C.c_char_p, []),
    "fd_setup": (C.c_int, [C.c_void_p, C.c_int, c_int64_p, C.POINTER(c_double_p), C.POINTER(c_double_p),
                           C.POINTER(FdSetupOpts), C.POINTER(C.c_void_p)]),
    "fd_setup_from_factors": (C.c_int, [C.c_void_p, C.c_int, c_int64_p, C.POINTER(c_double_p),
                                        C.POINTER(c_double_p), C.POINTER(c_double_p), C.POINTER(C.c_void_p)]),
    "fd_setup_from_blocks": (C.c_int, [C.c_void_p, C.c_int, c_int64_p, C.POINTER(c_double_p),
                                       C.POINTER(c_double_p), C.POINTER(c_double_p), C.POINTER(c_double_p),
                                       C.POINTER(C.c_void_p)]),
    "fd_setup_from_eig": (C.c_int, [C.c_void_p, C.c_int, c_int64_p, C.POINTER(c_double_p), C.POINTER(c_double_p),
                                    C.POINTER(c_double_p), C.POINTER(C.c_void_p)]),
    "fd_get_factors": (C.c_int, [C.c_void_p, C.c_int, c_double_p, c_double_p, c_double_p, c_double_p]),
    "fd_apply": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "fd_apply_host": (C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    "fd_apply_host_async": (C.c_int, [C.c_void_p, c_double_p, c_double_p]),
    "fd_host_sync": (C.c_int, [C.c_void_p]),
    "fd_apply_flops": (C.c_double, [C.c_void_p]),
    "fd_plan_path": (C.c_int, [C.c_void_p, c_double_p]),
    "fd_plan_set_path": (C.c_int, [C.c_void_p, C.c_int]),
    "fd_apply_timed": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(C.c_float), c_int32_p, C.c_int,
                                 C.POINTER(C.c_int)]),
    "fd_plan_destroy": (C.c_int, [C.c_void_p]),
    "stencil_create": (C.c_int, [C.c_void_p, C.c_int, c_int64_p, C.POINTER(c_int32_p), C.POINTER(c_int32_p),
                                 C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "colloc_assemble": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_int64_p, C.c_int, c_double_p,
                                  C.POINTER(C.c_void_p)]),
    "colloc_matrix_free": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_int64_p, C.c_int, c_double_p,
                                     C.POINTER(C.c_void_p)]),
    "colloc_assemble_cd": (C.c_int, [C.c_void_p, C.c_int, C.c_int, c_int64_p, C.c_int, c_double_p, C.c_int,
                                     c_double_p, C.c_int, C.POINTER(C.c_void_p)]),
    "colloc_1d_convection": (C.c_int, [C.c_int, C.c_int64, c_double_p, c_double_p]),
    "wq_assemble": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int64, C.c_int, c_double_p, C.POINTER(C.c_void_p)]),
    "galerkin_1d_factors": (C.c_int, [C.c_int, C.c_int64, c_double_p, c_double_p]),
    "stencil_matvec": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "stencil_info": (C.c_int, [C.c_void_p, c_int64_p, c_int64_p, c_int32_p, c_int32_p]),
    "stencil_get_values": (C.c_int, [C.c_void_p, c_double_p]),
    "stencil_destroy": (C.c_int, [C.c_void_p]),
    "colloc_1d_factors": (C.c_int, [C.c_int, C.c_int64, c_double_p, c_double_p]),
    "gmres_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.POINTER(GmresOpts),
                              C.POINTER(GmresReport)]),
    "bicgstab_solve": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                 C.POINTER(BicgstabOpts), C.POINTER(BicgstabReport)]),
    "fdiga_kernel_launches": (C.c_int64, [C.c_void_p]),
}

_lib = None


def load():
    """Load libfdiga.so (built in-tree).  Fails loudly: there is no fallback path."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"libfdiga.so not built at {LIB_PATH}; run `python __graft_entry__.py build` "
                              "(or paper_1705_04384_b200/build.py)")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


class FdigaError(RuntimeError):
    def __init__(self, status, where):
        lib = load()
        msg = lib.fdiga_last_error().decode(errors="replace")
        super().__init__(f"{where}: {lib.fdiga_status_string(status).decode()} ({status}): {msg}")
        self.status = status


def check(status, where):
    if status != 0:
        raise FdigaError(status, where)
    return status

"""C-ABI checks that need no GPU: the library loads, exports every entry point include/fdiga.h declares,
the Python binding declares the same set, and the host-only entry points work.  (no GPU)"""
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "fdiga.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\**\s+\**([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(names))


def test_header_declares_the_hot_path_calls():
    names = _declared()
    for required in ["fd_setup", "fd_apply", "stencil_matvec", "gmres_solve", "colloc_assemble",
                     "fd_setup_from_factors", "fdiga_ctx_create"]:
        assert required in names


def test_library_exports_every_declared_symbol():
    import ctypes
    from paper_1705_04384_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_covers_the_header():
    from paper_1705_04384_b200 import _lib
    assert sorted(_lib.SIGNATURES) == _declared()


def test_status_strings():
    from paper_1705_04384_b200 import load
    lib = load()
    assert lib.fdiga_status_string(0) == b"OK"
    assert lib.fdiga_status_string(-5) == b"COMPLEX_SPECTRUM"
    assert lib.fdiga_status_string(-8) == b"NOT_CONVERGED"


@pytest.mark.parametrize("ne,p", [(8, 2), (9, 3), (12, 5), (1, 3), (3, 1)])
def test_host_1d_factors_match_oracle(ne, p):
    # libfdiga's host spline tables (Piegl-Tiller in C++) vs the oracle's Cox-de Boor
    import paper_1705_04384_b200 as fd
    from oracle import splines
    M, K = fd.colloc_1d_factors(p, ne)
    _, Mo, Ko, _ = splines.colloc_1d(ne, p)
    np.testing.assert_allclose(M, Mo, rtol=0, atol=1e-14)
    np.testing.assert_allclose(K, Ko, rtol=0, atol=1e-12 * max(1, np.abs(Ko).max()))


def test_context_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import paper_1705_04384_b200 as fd
    with pytest.raises(fd.FdigaError):
        fd.Context(0)

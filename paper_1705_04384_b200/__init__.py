"""paper_1705_04384_b200 — B200-native FD-preconditioned GMRES for nonsymmetric IGA collocation.

The hot path (FD apply, stored-operator matvec, Arnoldi kernels) lives in libfdiga.so
(csrc/, C ABI in include/fdiga.h).  This package is its thin ctypes binding; it never falls back
to a CPU implementation: importing the API without the built library raises ImportError.
"""
from ._lib import LIB_PATH, FdigaError, load  # noqa: F401
from .api import (ORTH_CGS2, ORTH_DCGS2, bicgstab_solve, ORTH_CGS_DGKS, Context, FDPlan, LoopbackHub, Stencil, colloc_1d_factors,  # noqa: F401
                  colloc_1d_windows, colloc_1d_convection, wq_assemble, galerkin_1d_factors, halo_plan, transpose_plan,
                  colloc_assemble, fd_apply, fd_apply_timed, fd_apply_host, fd_apply_host_async, fd_host_sync, fd_setup, fd_setup_from_blocks, fd_setup_from_eig,
                  fd_setup_from_factors, gmres_solve, nccl_unique_id, partition, stencil_create,
                  stencil_matvec)

GEOM_IDENTITY, GEOM_ANNULUS, GEOM_DEFORMED_CUBE, GEOM_THICK_RING = 0, 1, 2, 3

"""CPU ORACLE — TEST INFRASTRUCTURE ONLY.

A plain, slow, obviously correct float64 CPU implementation of what the hot path
computes, written from the paper (/root/reference/PAPER.md, "P:<line>") and
independent of the CUDA library: it shares no code, headers, tables or constants
with `paper_1705_04384_b200/`, and neither imports the other.  Only `tests/`,
`__graft_entry__.smoke()` and `bench.py`'s cpu_baseline / `--impl reference` leg
may import it.  The product path never routes through it.

Modules
  splines   open knots, Cox-de Boor B-splines (+1st/2nd derivatives), Greville
            points, 1D collocation factors M^C, K^C
  geometry  analytic maps F with Jacobian J and Hessians H_c (configs)
  assembly  collocation operator A_C on a mapped domain: CSR assembly, the
            sum-factorised matvec, explicit single rows
  fastdiag  FD setup (generalized eig) and FD apply (loops, mode products), the
            dense Kronecker preconditioner P
  krylov    right-preconditioned restarted GMRES(m) with MGS (Saad 1986) and
            right-preconditioned BiCGStab with half-iteration accounting

Parity pins: every function is pinned by tests in tests/test_oracle_*.py against
values the paper or the mathematics fix (SPEC examples, closed forms, invariants,
brute force, finite-difference Laplacians, manufactured-solution convergence).
No function in this package is "parity unpinned".
"""

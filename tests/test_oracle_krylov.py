"""Pins for oracle/krylov.py GMRES(m) (no GPU): textbook properties and exact solves."""
import numpy as np
import pytest

from oracle import assembly, fastdiag, krylov
from synth import get_config, rhs


def test_identity_converges_in_one_iteration():
    b = np.random.default_rng(0).standard_normal(50)
    x, rep = krylov.gmres(lambda v: v.copy(), b)
    assert rep["iters"] == 1 and rep["converged"]
    np.testing.assert_allclose(x, b, atol=1e-14)


def test_minimal_polynomial_termination():
    # A diagonalizable with k distinct eigenvalues: GMRES terminates in exactly k steps (Saad 1986)
    rng = np.random.default_rng(1)
    vals = np.repeat([1.0, 2.0, 5.0, 7.0], 10)
    S = rng.standard_normal((40, 40)) + 8 * np.eye(40)
    A = S @ np.diag(vals) @ np.linalg.inv(S)
    b = rng.standard_normal(40)
    x, rep = krylov.gmres(lambda v: A @ v, b, rtol=1e-10)
    assert rep["iters"] == 4
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=1e-7)


@pytest.mark.parametrize("m", [30, 5])
def test_nonsymmetric_solve_matches_direct(m):
    rng = np.random.default_rng(2)
    n = 120
    A = np.eye(n) * 4 + rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    x, rep = krylov.gmres(lambda v: A @ v, b, m=m, rtol=1e-10, max_iters=2000)
    assert rep["converged"]
    assert rep["rel_res_true"] <= 1e-10 * 10
    np.testing.assert_allclose(x, np.linalg.solve(A, b), atol=1e-8)
    if m == 5:
        assert rep["restarts"] > 1
    # implicit and true residual agree within 10x
    assert rep["rel_res_true"] <= 10 * max(rep["rel_res_implicit"], 1e-10)


def test_exact_preconditioner_one_iteration():
    rng = np.random.default_rng(3)
    A = np.eye(30) * 3 + rng.standard_normal((30, 30)) * 0.3
    Ainv = np.linalg.inv(A)
    x, rep = krylov.gmres(lambda v: A @ v, rng.standard_normal(30), precond=lambda v: Ainv @ v)
    assert rep["iters"] == 1


def test_cfg1_fd_is_exact_solver():
    # identity map: A_C = P_C, so FD-preconditioned GMRES converges in one iteration
    c = get_config(1)
    disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
    f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
    x, rep = krylov.gmres(disc.matvec, rhs(1, disc.N), precond=lambda v: fastdiag.apply(f, v))
    assert rep["iters"] == 1 and rep["rel_res_true"] < 1e-12


def test_h_robust_iteration_counts():
    # iteration counts nearly independent of h
    counts = []
    for ne in (16, 32, 64):
        disc = assembly.Discretisation(2, 3, ne, 1, (1.0, 2.0))
        f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
        _, rep = krylov.gmres(disc.matvec, rhs(2, disc.N), precond=lambda v: fastdiag.apply(f, v))
        counts.append(rep["iters"])
    assert max(counts) - min(counts) <= 3 and max(counts) <= 35, counts

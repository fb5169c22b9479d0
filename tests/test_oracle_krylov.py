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


# ---- BiCGStab (the paper's solver) with half-iteration accounting

def test_bicgstab_identity_and_exact_preconditioner_half_iteration():
    # A = I: the first BiCG half step gives s = r - (r.r / r.r) r = 0 -> 0.5 iterations
    rng = np.random.default_rng(0)
    b = rng.standard_normal(40)
    x, rep = krylov.bicgstab(lambda v: v.copy(), b)
    assert rep["iters"] == 0.5 and rep["converged"]
    np.testing.assert_allclose(x, b, atol=1e-14)
    A = np.eye(30) * 3 + rng.standard_normal((30, 30)) * 0.3
    Ainv = np.linalg.inv(A)
    bb = rng.standard_normal(30)
    x, rep = krylov.bicgstab(lambda v: A @ v, bb, precond=lambda v: Ainv @ v)
    assert rep["iters"] == 0.5
    np.testing.assert_allclose(A @ x, bb, atol=1e-12)


def test_bicgstab_nonsymmetric_solve_matches_direct():
    rng = np.random.default_rng(2)
    n = 150
    A = np.eye(n) * 4 + rng.standard_normal((n, n)) / np.sqrt(n)
    b = rng.standard_normal(n)
    x, rep = krylov.bicgstab(lambda v: A @ v, b, rtol=1e-11)
    assert rep["converged"] and not rep["breakdown"]
    np.testing.assert_allclose(x, np.linalg.solve(A, b), atol=1e-9)
    # the recursive residual tracks the true one ("within 10x")
    assert rep["rel_res_true"] <= 10 * max(rep["rel_res_recursive"], 1e-12)
    # half-step accounting: a .5 count iff the last recorded residual is a BiCG half step
    assert (rep["iters"] % 1 == 0.5) == (len(rep["history"]) % 2 == 1)
    assert len(rep["history"]) == int(round(2 * rep["iters"]))


def test_bicgstab_breakdown_reported():
    # r^ . v = 0 at the first step: A a 90-degree rotation (r . A r = 0 for every r)
    A = np.array([[0.0, -1.0], [1.0, 0.0]])
    x, rep = krylov.bicgstab(lambda v: A @ v, np.array([1.0, 0.0]))
    assert rep["breakdown"] and not rep["converged"]


def test_bicgstab_cfg1_fd_exact():
    c = get_config(1)
    disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
    f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
    x, rep = krylov.bicgstab(disc.matvec, rhs(1, disc.N), precond=lambda v: fastdiag.apply(f, v))
    assert rep["iters"] == 0.5 and rep["rel_res_true"] < 1e-12


@pytest.mark.slow
def test_bicgstab_fd_counts_match_paper_table2():
    # Table 2: BiCGStab + FD on the quarter ring, collocation, 13.5 / 12.0 iterations, flat
    # in h and p.  The paper leaves radii, f and the tolerance unstated: with radii 1, 2, Matlab's
    # default bicgstab tolerance 1e-6 and x0 = 0 (DESIGN.md readings), both a random b and f = 1 land
    # within 2 half-iterations of every printed cell for h^-1 = 128, 256.
    import json
    import os
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_table2_bicgstab.json")))
    for ne in (128, 256):
        for j, p in enumerate(gold["p"]):
            disc = assembly.Discretisation(2, p, ne, 1, (1.0, 2.0))
            f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
            for b in (rhs(2, disc.N), np.ones(disc.N)):
                _, rep = krylov.bicgstab(disc.matvec, b, precond=lambda v: fastdiag.apply(f, v), rtol=1e-6)
                assert rep["converged"]
                assert abs(rep["iters"] - gold["iterations"][str(ne)][j]) <= 2.0, (ne, p, rep["iters"])

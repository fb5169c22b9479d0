"""Pins for oracle/fastdiag.py (no GPU).

  * SPEC.md:414 / SPEC.md:423 worked examples (tests/golden/spec_examples.json)
  * brute force on tiny n: P s = b and P^{-1}(P v) = v with P materialised by np.kron (eq:colloc2D/3D)
  * the explicit-loop apply equals the mode-product apply (eq:FD2D / eq:FD3D written two ways)
  * setup residuals K U = M U D and W M U = I, Remark 1 real spectrum
  * low pencil eigenvalues approach the Dirichlet Laplacian eigenvalues k^2 pi^2 on [0,1] (closed form)
  * flop model 12 n^4 and 8 n^3
"""
import json
import os

import numpy as np
import pytest

from oracle import assembly, fastdiag, splines

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def test_spec_worked_apply_example():
    ex = GOLD["fd_apply"][0]
    M, K = np.array(ex["M"], float), np.array(ex["K"], float)
    f = fastdiag.setup([M] * ex["d"], [K] * ex["d"])
    np.testing.assert_allclose(fastdiag.apply(f, np.array(ex["b"], float)), ex["s"], atol=1e-15)
    np.testing.assert_allclose(fastdiag.apply_loops(f, np.array(ex["b"], float)), ex["s"], atol=1e-15)


def test_spec_setup_example():
    ex = GOLD["fd_setup"][0]
    U, W, lam = fastdiag.setup_direction(np.array(ex["M"], float), np.array(ex["K"], float))
    np.testing.assert_allclose(lam, ex["lam"], atol=1e-15)
    np.testing.assert_allclose(np.abs(U), ex["U_abs"], atol=1e-15)
    np.testing.assert_allclose(np.abs(W.T), ex["V_abs"], atol=1e-15)


@pytest.mark.parametrize("d,ne,p", [(2, 4, 2), (2, 5, 3), (3, 3, 3), (3, 4, 2)])
def test_brute_force_inverse_of_kron_preconditioner(d, ne, p):
    tau, M, K, _ = splines.colloc_1d(ne, p)
    f = fastdiag.setup([M] * d, [K] * d)
    P = assembly.kron_preconditioner_dense([M] * d, [K] * d)
    rng = np.random.default_rng(11)
    for _ in range(5):
        b = rng.standard_normal(P.shape[0])
        s = fastdiag.apply(f, b)
        assert np.linalg.norm(P @ s - b) / np.linalg.norm(b) < 1e-12
        v = rng.standard_normal(P.shape[0])
        assert np.linalg.norm(fastdiag.apply(f, P @ v) - v) / np.linalg.norm(v) < 1e-12
        np.testing.assert_allclose(fastdiag.apply_loops(f, b), s, atol=1e-12 * np.abs(s).max())
        # the plain definition s = P^{-1} b (dense LU)
        np.testing.assert_allclose(s, np.linalg.solve(P, b), atol=1e-11 * np.abs(s).max())


def test_anisotropic_factor_sizes():
    # different n_l per direction: checks that factor l acts on index i_l
    rng = np.random.default_rng(5)
    ns = [3, 4, 5]
    U = [rng.standard_normal((n, n)) + 3 * np.eye(n) for n in ns]
    lam = [rng.uniform(1, 10, n) for n in ns]
    f = fastdiag.factors_from_eig(U, lam)
    # P = sum_k (x)_{l=3..1} (K_l if l==k else M_l), M_l = V^{-T} U^{-1} = I (W = U^{-1}), K_l = U D U^{-1}
    Ms = [np.eye(n) for n in ns]
    Ks = [U[l] @ np.diag(lam[l]) @ np.linalg.inv(U[l]) for l in range(3)]
    P = assembly.kron_preconditioner_dense(Ms, Ks)
    b = rng.standard_normal(P.shape[0])
    np.testing.assert_allclose(P @ fastdiag.apply(f, b), b, atol=1e-10)
    np.testing.assert_allclose(fastdiag.apply_loops(f, b), fastdiag.apply(f, b), atol=1e-12)


@pytest.mark.parametrize("ne,p", [(32, 2), (64, 3), (16, 5)])
def test_setup_residuals_and_remark1(ne, p):
    _, M, K, _ = splines.colloc_1d(ne, p)
    U, W, lam = fastdiag.setup_direction(M, K)
    assert np.linalg.norm(K @ U - M @ U @ np.diag(lam)) / (np.linalg.norm(K) * np.linalg.norm(U)) < 1e-13
    assert np.linalg.norm(W @ M @ U - np.eye(len(lam))) < 1e-11
    assert np.all(np.diff(lam) >= 0) and lam[0] > 0
    np.testing.assert_allclose(np.linalg.norm(U, axis=0), 1.0, atol=1e-14)


def test_low_eigenvalues_approach_dirichlet_laplacian():
    # -u'' = lam u on (0,1), u(0)=u(1)=0: lam_k = k^2 pi^2.  The pencil (K^C, M^C) discretises it.
    _, M, K, _ = splines.colloc_1d(128, 5)
    _, _, lam = fastdiag.setup_direction(M, K)
    exact = np.array([1, 4, 9]) * np.pi ** 2
    np.testing.assert_allclose(lam[:3], exact, rtol=1e-6)


def test_flop_model():
    assert fastdiag.flops([256] * 3) == 12 * 256 ** 4
    assert fastdiag.flops([100] * 2) == 8 * 100 ** 3

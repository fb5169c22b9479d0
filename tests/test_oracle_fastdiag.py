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
    U, W, lam, _ = fastdiag.setup_direction(np.array(ex["M"], float), np.array(ex["K"], float))
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
    U, W, lam, _ = fastdiag.setup_direction(M, K)
    assert np.linalg.norm(K @ U - M @ U @ np.diag(lam)) / (np.linalg.norm(K) * np.linalg.norm(U)) < 1e-13
    assert np.linalg.norm(W @ M @ U - np.eye(len(lam))) < 1e-11
    assert np.all(np.diff(lam) >= 0) and lam[0] > 0
    np.testing.assert_allclose(np.linalg.norm(U, axis=0), 1.0, atol=1e-14)


def test_low_eigenvalues_approach_dirichlet_laplacian():
    # -u'' = lam u on (0,1), u(0)=u(1)=0: lam_k = k^2 pi^2.  The pencil (K^C, M^C) discretises it.
    _, M, K, _ = splines.colloc_1d(128, 5)
    _, _, lam, _ = fastdiag.setup_direction(M, K)
    exact = np.array([1, 4, 9]) * np.pi ** 2
    np.testing.assert_allclose(lam[:3], exact, rtol=1e-6)


def test_flop_model():
    assert fastdiag.flops([256] * 3) == 12 * 256 ** 4
    assert fastdiag.flops([100] * 2) == 8 * 100 ** 3


# ---- complex pairs in real 2x2-block form

def test_galerkin_factors_pins():
    # exact integrals: full-basis row sums of M are int B_i = (xi_{i+p+1} - xi_i)/(p+1); for interior
    # functions H + H^T = [B_i B_j]_0^1 = 0 (constant wind); K is symmetric positive definite
    ne, p, w = 6, 2, 3.0
    M, K, H = splines.galerkin_1d(ne, p, w)
    kv = splines.open_uniform_knots(ne, p)
    n = M.shape[0]
    np.testing.assert_allclose(M, M.T, atol=1e-15)
    np.testing.assert_allclose(H + H.T, 0.0, atol=1e-13)
    assert np.all(np.linalg.eigvalsh(K) > 0)
    # sum_j M_ij over the interior j equals int B_i minus the two boundary-function overlaps; check a
    # middle row, which overlaps no boundary function
    i = n // 2
    np.testing.assert_allclose(M[i].sum(), (kv[i + 1 + p + 1] - kv[i + 1]) / (p + 1), rtol=1e-13)


def test_convection_diffusion_pencil_has_complex_pairs():
    # eq:convec_prec_2 with a strong constant wind: all eigenvalues of (K + H, M) complex
    M, K, H = splines.galerkin_1d(32, 2, 100.0)
    with pytest.raises(ValueError):
        fastdiag.setup_direction(M, K + H)
    U, W, lam, lam_im = fastdiag.setup_direction(M, K + H, allow_complex=True)
    assert np.count_nonzero(lam_im) == 32
    f = fastdiag.FDFactors([U], [W], [lam], [lam_im])
    D = f.D(0)
    # M^{-1}(K+H) U = U D with the real 2x2 blocks [[a, b], [-b, a]]
    np.testing.assert_allclose(np.linalg.solve(M, K + H) @ U, U @ D, atol=1e-9 * np.abs(D).max())
    np.testing.assert_allclose(W @ M @ U, np.eye(32), atol=1e-10)


@pytest.mark.parametrize("d,wind,ne", [(2, 100.0, 6), (3, 100.0, 4), (2, 30.0, 7), (3, 60.0, 5)])
def test_complex_pair_apply_is_exact_solver(d, wind, ne):
    # mixed real / complex spectra (moderate wind) and all-complex spectra; P s = b by brute force
    M, K, H = splines.galerkin_1d(ne, 2, wind)
    f = fastdiag.setup([M] * d, [K + H] * d, allow_complex=True)
    assert f.has_pairs
    P = assembly.kron_preconditioner_dense([M] * d, [K + H] * d)
    rng = np.random.default_rng(d)
    b = rng.standard_normal(P.shape[0])
    s = fastdiag.apply(f, b)
    np.testing.assert_allclose(s, np.linalg.solve(P, b), atol=1e-10 * np.abs(s).max())


def test_complex_pair_rotation_blocks_closed_form():
    # M = I, K = rotation-scaling blocks: eigenvalues 2 +- 3i and 5; Lambda^{-1} on one block is a 2x2
    # inverse, so for d = 2 the apply must equal the dense solve of K (x) I + I (x) K
    K = np.array([[2.0, 3.0, 0.0], [-3.0, 2.0, 0.0], [0.0, 0.0, 5.0]])
    f = fastdiag.setup([np.eye(3)] * 2, [K] * 2, allow_complex=True)
    P = np.kron(K, np.eye(3)) + np.kron(np.eye(3), K)
    b = np.arange(1.0, 10.0)
    np.testing.assert_allclose(fastdiag.apply(f, b), np.linalg.solve(P, b), atol=1e-13)

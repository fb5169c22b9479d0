"""Pins for oracle/quadrature.py (NEXT-3, weighted quadrature; no GPU)."""
import json
import os

import numpy as np
import pytest

from oracle import assembly, quadrature as qd, splines
from synth.configs import GEOM_ANNULUS, GEOM_IDENTITY, GEOM_THICK_RING

GOLD_EH = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_table1_eh.json")))


def test_gauss_rule_spec_examples():
    # 1 point on [0,1] -> 0.5 / 1; 2 points -> 0.5 -+ 1/(2 sqrt 3), weights 0.5; x^3 exactly
    x, w = qd.gauss_rule(1, 0, 1)
    np.testing.assert_allclose([x[0], w[0]], [0.5, 1.0], atol=1e-15)
    x, w = qd.gauss_rule(1, 1, 2)
    np.testing.assert_allclose(np.sort(x), [0.5 - 1 / (2 * np.sqrt(3)), 0.5 + 1 / (2 * np.sqrt(3))], atol=1e-15)
    np.testing.assert_allclose(w, [0.5, 0.5], atol=1e-15)
    np.testing.assert_allclose(np.sum(w * x ** 3), 0.25, atol=1e-15)


@pytest.mark.parametrize("ne,p", [(6, 2), (7, 3), (8, 4), (9, 5), (2, 2)])
def test_wq_exactness_against_independent_galerkin_factors(ne, p):
    # sum_q w^{ab}_{iq} B_j^{(b)}(x_q) = int B_i^{(a)} B_j^{(b)}: compared with splines.galerkin_1d (its own
    # Gauss loop): M (a=b=0), K (a=b=1), H (a=0, b=1, unit wind) and H^T (a=1, b=0)
    xq, W, E = qd.wq_rule_1d(ne, p)
    M, K, H = splines.galerkin_1d(ne, p, 1.0)
    for (a, b), ref in {(0, 0): M, (1, 1): K, (0, 1): H, (1, 0): H.T}.items():
        got = W[(a, b)] @ E[b]
        band = np.abs(np.subtract.outer(np.arange(len(M)), np.arange(len(M)))) <= p
        np.testing.assert_allclose(got[band], ref[band], atol=1e-12 * max(1.0, np.abs(ref).max()))


@pytest.mark.parametrize("p", [2, 3, 4, 5])
def test_wq_points_per_row_are_order_p(p):
    # SPEC quadrature invariant: O(p) points per row (2p + 3 for interior rows)
    ne = 12
    xq, W, E = qd.wq_rule_1d(ne, p)
    counts = (np.abs(W[(1, 1)]) > 0).sum(axis=1)
    assert counts.max() <= 2 * p + 3 + 4 and np.median(counts) <= 2 * p + 3


@pytest.mark.parametrize("d,p,ne", [(2, 2, 5), (2, 3, 6), (3, 2, 3), (3, 3, 4)])
def test_wq_identity_map_is_exact_kronecker(d, p, ne):
    # P:204-214 (eq:wq2D / eq:wq3D): on the identity map WQ is exact and A_wq is the Kronecker form of the
    # exact Galerkin factors (eq:univariateWQ), symmetric positive definite
    disc = qd.WQDiscretisation(d, p, ne, GEOM_IDENTITY)
    A = disc.assemble_wq().toarray()
    M, K, _ = splines.galerkin_1d(ne, p, 0.0)
    P = assembly.kron_preconditioner_dense([M] * d, [K] * d)
    np.testing.assert_allclose(A, P, atol=1e-12 * np.abs(P).max())
    np.testing.assert_allclose(disc.assemble_galerkin().toarray(), P, atol=1e-12 * np.abs(P).max())


def test_wq_mapped_domain_nonsymmetric_and_close_to_galerkin():
    # A_wq is in general nonsymmetric; it approximates A_G
    disc = qd.WQDiscretisation(2, 3, 8, GEOM_ANNULUS, (1.0, 2.0))
    A = disc.assemble_wq().toarray()
    G = disc.assemble_galerkin().toarray()
    assert np.abs(A - A.T).max() > 1e-6 * np.abs(A).max()
    np.testing.assert_allclose(G, G.T, atol=1e-12 * np.abs(G).max())
    assert np.linalg.norm(A - G) / np.linalg.norm(G) < 0.05


@pytest.mark.parametrize("p", [2, 3])
def test_eh_matches_paper_table1(p):
    # Table 1: e_h = ||H^{-1/2}(A_wq - A_G)H^{-1/2}||, quarter ring; radii 1, 2 (reading 8/9):
    # within 15% of every printed value for h = 1/8, 1/16, 1/32, and e_h = O(h) (ratio ~2 per halving)
    vals = [qd.e_h(qd.WQDiscretisation(2, p, ne, GEOM_ANNULUS, (1.0, 2.0))) for ne in (8, 16, 32)]
    ref = GOLD_EH["e_h"][str(p)][:3]
    for v, r in zip(vals, ref):
        assert abs(v / r - 1) <= 0.15, (p, vals, ref)
    for a, b in zip(vals, vals[1:]):
        assert 1.8 <= a / b <= 2.1


def test_eh_is_order_h_for_even_p():
    # p = 4: the boundary rows use the extra points of reading 18 -- still e_h = O(h)
    vals = [qd.e_h(qd.WQDiscretisation(2, 4, ne, GEOM_ANNULUS, (1.0, 2.0))) for ne in (8, 16)]
    assert 1.8 <= vals[0] / vals[1] <= 2.1


def test_wq_3d_thick_ring_close_to_galerkin():
    disc = qd.WQDiscretisation(3, 2, 4, GEOM_THICK_RING, (1.0, 2.0, 1.0))
    A = disc.assemble_wq().toarray()
    G = disc.assemble_galerkin().toarray()
    assert np.linalg.norm(A - G) / np.linalg.norm(G) < 0.05


@pytest.mark.slow
def test_wq_bicgstab_counts_match_paper_table3():
    # Table 3: BiCGStab + FD on the WQ quarter ring needs 16.0 iterations for every h and p; with the
    # readings of Table 2's pin (radii 1, 2, tol 1e-6, x0 = 0) and a random b the counts are within 2 and
    # independent of p (the preconditioner is the symmetric FD of the exact Galerkin pencils)
    from oracle import fastdiag, krylov
    from synth import rhs
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_table3_wq_bicgstab.json")))
    counts = []
    for j, p in enumerate(gold["p"]):
        disc = qd.WQDiscretisation(2, p, 128, GEOM_ANNULUS, (1.0, 2.0))
        A = disc.assemble_wq()
        M, K, _ = splines.galerkin_1d(128, p, 0.0)
        f = fastdiag.setup([M] * 2, [K] * 2)
        _, rep = krylov.bicgstab(lambda v: A @ v, rhs(8, disc.N), precond=lambda v: fastdiag.apply(f, v), rtol=1e-6)
        assert rep["converged"] and abs(rep["iters"] - gold["iterations"]["128"][j]) <= 2.0
        counts.append(rep["iters"])
    assert max(counts) - min(counts) <= 1.0

"""Pins for oracle/splines.py against values the paper/SPEC print and closed forms (no GPU)."""
import json
import os

import numpy as np
import pytest

from oracle import splines

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.mark.parametrize("ex", GOLD["knots"])
def test_knots_spec_examples(ex):
    kv = splines.open_uniform_knots(ex["ne"], ex["p"])
    m = len(kv) - ex["p"] - 1
    assert m == ex["m"]
    if "knots" in ex:
        np.testing.assert_array_equal(kv, ex["knots"])
    else:
        np.testing.assert_allclose(kv[ex["p"] + 1:-(ex["p"] + 1)], ex["interior"], rtol=0, atol=0)


@pytest.mark.parametrize("ex", GOLD["basis"])
def test_basis_spec_examples(ex):
    vals = splines.basis_all(np.array(ex["knots"], float), ex["p"], ex["x"], ex["deriv"])
    np.testing.assert_allclose(vals, ex["values"], atol=1e-15)


@pytest.mark.parametrize("ex", GOLD["greville"])
def test_greville_spec_examples(ex):
    np.testing.assert_allclose(splines.greville_interior(np.array(ex["knots"], float), ex["p"]), ex["tau"],
                               atol=1e-15)


@pytest.mark.parametrize("ex", GOLD["flatten"])
def test_flatten_spec_examples(ex):
    assert splines.flatten_index(ex["mi"], ex["n"]) == ex["i"]


@pytest.mark.parametrize("p", [2, 3])
def test_bernstein_closed_form(p):
    # one element: the B-splines are the Bernstein polynomials C(p,k) x^k (1-x)^(p-k)
    from math import comb
    kv = np.array([0.0] * (p + 1) + [1.0] * (p + 1))
    for x in [0.0, 0.13, 0.5, 0.77, 1.0]:
        b0 = [comb(p, k) * x ** k * (1 - x) ** (p - k) for k in range(p + 1)]
        # derivatives by the closed form d/dx x^k (1-x)^(p-k)
        def d1(k):
            t1 = k * x ** (k - 1) * (1 - x) ** (p - k) if k > 0 else 0.0
            t2 = -(p - k) * x ** k * (1 - x) ** (p - k - 1) if p - k > 0 else 0.0
            return comb(p, k) * (t1 + t2)

        def d2(k):
            a = k * (k - 1) * x ** (k - 2) * (1 - x) ** (p - k) if k > 1 else 0.0
            b = -2 * k * (p - k) * x ** (k - 1) * (1 - x) ** (p - k - 1) if (k > 0 and p - k > 0) else 0.0
            c = (p - k) * (p - k - 1) * x ** k * (1 - x) ** (p - k - 2) if p - k > 1 else 0.0
            return comb(p, k) * (a + b + c)
        np.testing.assert_allclose(splines.basis_all(kv, p, x, 0), b0, atol=1e-14)
        np.testing.assert_allclose(splines.basis_all(kv, p, x, 1), [d1(k) for k in range(p + 1)], atol=1e-13)
        np.testing.assert_allclose(splines.basis_all(kv, p, x, 2), [d2(k) for k in range(p + 1)], atol=1e-12)


@pytest.mark.parametrize("ne,p", [(5, 2), (7, 3), (6, 5)])
def test_partition_of_unity_support_greville_reproduction(ne, p):
    kv = splines.open_uniform_knots(ne, p)
    g = splines.greville_full(kv, p)
    rng = np.random.default_rng(0)
    for x in list(rng.uniform(0, 1, 25)) + [0.0, 1.0, 1.0 / ne]:
        B = splines.basis_all(kv, p, x, 0)
        assert abs(B.sum() - 1.0) < 1e-12
        assert np.count_nonzero(np.abs(B) > 0) <= p + 1
        assert abs(g @ B - x) < 1e-12
        assert abs(splines.basis_all(kv, p, x, 1).sum()) < 1e-9
        assert abs(splines.basis_all(kv, p, x, 2).sum()) < 1e-7


@pytest.mark.parametrize("ne,p", [(6, 3), (5, 4)])
def test_derivatives_match_finite_differences(ne, p):
    kv = splines.open_uniform_knots(ne, p)
    h = 1e-6
    rng = np.random.default_rng(1)
    for x in rng.uniform(0.01, 0.99, 10):
        for r in (0, 1):
            fd = (splines.basis_all(kv, p, x + h, r) - splines.basis_all(kv, p, x - h, r)) / (2 * h)
            np.testing.assert_allclose(splines.basis_all(kv, p, x, r + 1), fd, atol=1e-5 * max(1, ne ** (r + 1)))


def test_greville_strictly_increasing_interior():
    for ne, p in [(4, 3), (32, 2), (64, 3), (8, 5)]:
        tau = splines.greville_interior(splines.open_uniform_knots(ne, p), p)
        assert len(tau) == ne + p - 2
        assert np.all(np.diff(tau) > 0) and tau[0] > 0 and tau[-1] < 1


@pytest.mark.parametrize("ne,p", [(8, 2), (9, 3), (7, 4), (10, 5)])
def test_colloc_1d_interpolates_polynomial(ne, p):
    # u(x) = x(1-x) lies in the interior spline space for p >= 2 (it vanishes at 0 and 1);
    # its coefficients c solve M c = u(tau); then K c = -u''(tau) = 2 exactly.
    tau, M, K, D1 = splines.colloc_1d(ne, p)
    c = np.linalg.solve(M, tau * (1 - tau))
    np.testing.assert_allclose(K @ c, 2.0, rtol=0, atol=1e-10)
    np.testing.assert_allclose(D1 @ c, 1 - 2 * tau, atol=1e-11)


def test_colloc_1d_full_basis_row_sums():
    # sum_j B_j = 1 and sum_j B_j'' = 0 over the FULL basis
    ne, p = 12, 3
    kv = splines.open_uniform_knots(ne, p)
    tau = splines.greville_interior(kv, p)
    for t in tau:
        assert abs(splines.basis_all(kv, p, t, 0).sum() - 1) < 1e-13
        assert abs(splines.basis_all(kv, p, t, 2).sum()) < 1e-9

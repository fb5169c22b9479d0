"""Pins for oracle/assembly.py + oracle/geometry.py (no GPU).

  * identity map, K = I: A_C equals the Kronecker forms eq:colloc2D / eq:colloc3D
  * every entry (A_C)_{ij} equals -Laplacian_x of B^_j o F^{-1} at F(tau_i), computed by finite
    differences in physical space through the inverse map (independent of the chain-rule formula)
  * manufactured solutions: the collocation error at the Greville points decays under h-halving
  * the CSR, sum-factorised and explicit-row formulations agree
"""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

from oracle import assembly, geometry as geo, splines
from synth.configs import GEOM_ANNULUS, GEOM_DEFORMED_CUBE, GEOM_IDENTITY, GEOM_THICK_RING


@pytest.mark.parametrize("d,p,ne", [(2, 2, 6), (2, 3, 5), (3, 3, 4), (3, 2, 4)])
def test_identity_map_is_kronecker_form(d, p, ne):
    disc = assembly.Discretisation(d, p, ne, GEOM_IDENTITY)
    A = disc.assemble_csr().toarray()
    P = assembly.kron_preconditioner_dense([disc.M] * d, [disc.K] * d)
    np.testing.assert_allclose(A, P, atol=1e-12 * np.abs(P).max())


def _fd_laplacian_entry(disc, i_flat, j_flat, h=1e-4):
    """-Lap_x (B^_j o F^{-1}) at x0 = F(tau_i) by the (2d+1)-point central stencil."""
    d, n = disc.d, disc.n
    kv = splines.open_uniform_knots(disc.ne, disc.p)
    ii = [(i_flat // n ** l) % n for l in range(d)]
    jj = [(j_flat // n ** l) % n for l in range(d)]
    xi0 = np.array([[disc.tau[ii[l]] for l in range(d)]])
    x0, _, _ = geo.evaluate(disc.geometry, xi0, disc.params)

    def u(x):
        xi = geo.inverse(disc.geometry, x[None, :], disc.params)[0]
        v = 1.0
        for l in range(d):
            v *= splines.basis_all(kv, disc.p, float(np.clip(xi[l], 0, 1)), 0)[jj[l] + 1]
        return v

    lap = 0.0
    c = u(x0[0])
    for k in range(d):
        e = np.zeros(d)
        e[k] = h
        lap += (u(x0[0] + e) - 2 * c + u(x0[0] - e)) / h ** 2
    return -lap


@pytest.mark.parametrize("d,geom,params", [(2, GEOM_ANNULUS, (1.0, 2.0)),
                                           (3, GEOM_DEFORMED_CUBE, (0.1,)),
                                           (3, GEOM_THICK_RING, (1.0, 2.0, 1.0))])
def test_entries_equal_physical_laplacian(d, geom, params):
    # p = 5 so that B^ o F^{-1} is C^4 and the central difference error is O(h^2)
    disc = assembly.Discretisation(d, 5, 5, geom, params)
    rng = np.random.default_rng(7)
    n = disc.n
    rows = rng.choice(disc.N, 3, replace=False)
    checked = 0
    for i in rows:
        row = disc.row(int(i))
        scale = max(abs(v) for v in row.values())
        for j, v in list(row.items())[:6]:
            fd = _fd_laplacian_entry(disc, int(i), j)
            assert abs(fd - v) <= 2e-4 * scale, (i, j, v, fd)
            checked += 1
    assert checked >= 9


def test_three_formulations_agree():
    disc = assembly.Discretisation(3, 3, 5, GEOM_DEFORMED_CUBE, (0.1,))
    A = disc.assemble_csr()
    x = np.random.default_rng(3).standard_normal(disc.N)
    y = A @ x
    np.testing.assert_allclose(disc.matvec(x), y, atol=1e-12 * np.abs(y).max())
    for i in [0, 17, disc.N // 2, disc.N - 1]:
        row = disc.row(i)
        dense = A[i].toarray()[0]
        for j, v in row.items():
            assert abs(dense[j] - v) <= 1e-12 * np.abs(dense).max()
        assert set(np.nonzero(dense)[0]) <= set(row)


def _manufactured(geom):
    if geom == GEOM_ANNULUS:
        def u(x):
            s = x[:, 0] ** 2 + x[:, 1] ** 2
            return (s - 1) * (s - 4) * x[:, 0] * x[:, 1]

        def f(x):   # -Lap u = xy(60 - 32 s)   (hand derivation in DESIGN.md)
            s = x[:, 0] ** 2 + x[:, 1] ** 2
            return x[:, 0] * x[:, 1] * (60 - 32 * s)
        return u, f, (1.0, 2.0)
    if geom == GEOM_DEFORMED_CUBE:   # the map fixes the boundary, so Omega = [0,1]^3
        def u(x):
            return np.prod(np.sin(np.pi * x), axis=1)

        def f(x):
            return 3 * np.pi ** 2 * np.prod(np.sin(np.pi * x), axis=1)
        return u, f, (0.1,)
    if geom == GEOM_THICK_RING:
        def u(x):
            s = x[:, 0] ** 2 + x[:, 1] ** 2
            return (s - 1) * (s - 4) * x[:, 0] * x[:, 1] * x[:, 2] * (1 - x[:, 2])

        def f(x):
            s = x[:, 0] ** 2 + x[:, 1] ** 2
            q = (s - 1) * (s - 4) * x[:, 0] * x[:, 1]
            z = x[:, 2]
            return z * (1 - z) * x[:, 0] * x[:, 1] * (60 - 32 * s) + 2 * q
        return u, f, (1.0, 2.0, 1.0)


@pytest.mark.parametrize("d,p,geom,nes", [(2, 3, GEOM_ANNULUS, (8, 16, 32)),
                                           (2, 4, GEOM_ANNULUS, (8, 16, 32)),
                                           (3, 3, GEOM_DEFORMED_CUBE, (4, 8, 16)),
                                           (3, 3, GEOM_THICK_RING, (4, 8, 16))])
def test_manufactured_solution_error_decays(d, p, geom, nes):
    u, f, params = _manufactured(geom)
    errs = []
    for ne in nes:
        disc = assembly.Discretisation(d, p, ne, geom, params)
        xphys, _, _ = geo.evaluate(geom, disc.points(), params)
        coef = spla.spsolve(disc.assemble_csr().tocsc(), f(xphys))
        # u_h(F(tau)) = sum_j c_j B^_j(tau) = (M_d (x) ... (x) M_1) c
        Mk = disc.kron_factor((0,) * d)
        errs.append(np.abs(Mk @ coef - u(xphys)).max() / np.abs(u(xphys)).max())
    ratios = [errs[k] / errs[k + 1] for k in range(len(errs) - 1)]
    assert errs[-1] < 1e-2
    assert min(ratios) > 2.5, (errs, ratios)


def test_chain_rule_coefficients_identity():
    disc = assembly.Discretisation(2, 3, 4, GEOM_IDENTITY)
    G, beta = disc.coefficients()
    np.testing.assert_allclose(G, np.broadcast_to(np.eye(2), G.shape), atol=0)
    np.testing.assert_allclose(beta, 0, atol=0)


# ---- convection-diffusion (NEXT-4; eq:convection P:345, L_w = -Lap + w . grad)

def test_convection_identity_map_constant_wind_is_kronecker():
    # identity map, constant wind: A = sum_k (x)_l (K_k + H_k if l = k else M_l) with the collocation
    # factor H_k = w_k B'_j(tau_i) (the collocation analogue of eq:convec_prec_2)
    d, p, ne, w = 3, 3, 4, (2.0, -3.0, 0.5)
    disc = assembly.Discretisation(d, p, ne, GEOM_IDENTITY, (), wind=geo.WIND_CONSTANT, wind_params=w)
    A = disc.assemble_csr().toarray()
    Ks = [disc.K + splines.colloc_1d_convection(ne, p, w[l]) for l in range(d)]
    P = assembly.kron_preconditioner_dense([disc.M] * d, Ks)
    np.testing.assert_allclose(A, P, atol=1e-12 * np.abs(P).max())


def test_convection_factor_pins():
    # full-basis derivative rows sum to 0 (partition of unity); Greville reproduction x = sum tau*_j B_j
    # differentiates to sum_j tau*_j B'_j = 1, so on interior rows far from the boundary H reproduces w~
    ne, p = 8, 3
    knots = splines.open_uniform_knots(ne, p)
    tau_full = splines.greville_full(knots, p)
    tau, M, K, D1 = splines.colloc_1d(ne, p)
    H = splines.colloc_1d_convection(ne, p, 5.0)
    np.testing.assert_allclose(H, 5.0 * D1, atol=0)
    i = len(tau) // 2
    row_full = np.array([splines.basis_all(knots, p, tau[i], 1)[k] for k in range(len(tau_full))])
    np.testing.assert_allclose(row_full.sum(), 0.0, atol=1e-12)
    np.testing.assert_allclose(row_full @ tau_full, 1.0, atol=1e-12)


def _fd_convection_entry(disc, i_flat, j_flat, h=1e-4):
    """(-Lap + w . grad)(B^_j o F^{-1}) at F(tau_i) by central differences in physical space."""
    d, n = disc.d, disc.n
    kv = splines.open_uniform_knots(disc.ne, disc.p)
    ii = [(i_flat // n ** l) % n for l in range(d)]
    jj = [(j_flat // n ** l) % n for l in range(d)]
    xi0 = np.array([[disc.tau[ii[l]] for l in range(d)]])
    x0, _, _ = geo.evaluate(disc.geometry, xi0, disc.params)

    def u(x):
        xi = geo.inverse(disc.geometry, x[None, :], disc.params)[0]
        v = 1.0
        for l in range(d):
            v *= splines.basis_all(kv, disc.p, float(np.clip(xi[l], 0, 1)), 0)[jj[l] + 1]
        return v

    c = u(x0[0])
    w = geo.wind(disc.wind, x0, disc.wind_params)[0]
    val = 0.0
    for k in range(d):
        e = np.zeros(d)
        e[k] = h
        up, um = u(x0[0] + e), u(x0[0] - e)
        val += -(up - 2 * c + um) / h ** 2 + w[k] * (up - um) / (2 * h)
    return val


@pytest.mark.parametrize("d,geom,params,wind,wp", [(2, GEOM_ANNULUS, (1.0, 2.0), geo.WIND_ROTATING, (7.0,)),
                                                   (3, GEOM_THICK_RING, (1.0, 2.0, 1.0), geo.WIND_ROTATING, (3.0,)),
                                                   (3, GEOM_DEFORMED_CUBE, (0.1,), geo.WIND_CONSTANT,
                                                    (1.0, -2.0, 4.0))])
def test_convection_entries_equal_physical_operator(d, geom, params, wind, wp):
    disc = assembly.Discretisation(d, 5, 5, geom, params, wind=wind, wind_params=wp)
    rng = np.random.default_rng(11)
    for i in rng.choice(disc.N, 3, replace=False):
        row = disc.row(int(i))
        for j in list(row)[:6]:
            ref = _fd_convection_entry(disc, int(i), int(j))
            assert abs(row[j] - ref) <= 2e-5 * max(1.0, abs(ref)), (i, j, row[j], ref)


def test_rotating_wind_is_angular_on_the_ring():
    # w = omega (-y, x, 0) on the thick ring: J^{-1} w = (0, 2 omega / pi, 0) exactly (synth NEXT-4 configs)
    xi = np.random.default_rng(2).uniform(0, 1, (20, 3))
    F, J, _ = geo.thick_ring(xi)
    v = np.linalg.solve(J, geo.wind(geo.WIND_ROTATING, F, (3.0,))[..., None])[..., 0]
    np.testing.assert_allclose(v, np.tile([0.0, 6.0 / np.pi, 0.0], (20, 1)), atol=1e-12)


@pytest.mark.parametrize("ns", [(2, 3), (3, 2), (2, 3, 4), (4, 3, 2), (3, 1, 2)])
def test_kron_preconditioner_builders_match_entrywise_definition(ns):
    # P = sum_k (x)_{l=d..1} (K_l if l == k else M_l) with i_1 fastest, written
    # out entry by entry: P[i, j] = sum_k prod_l A^{(k)}_l[i_l, j_l].  Anisotropic sizes and distinct random
    # factors per direction, so a swapped Kronecker order or a factor acting on the wrong index fails.
    rng = np.random.default_rng(sum(ns) * 7 + len(ns))
    d = len(ns)
    Ms = [rng.standard_normal((n, n)) for n in ns]
    Ks = [rng.standard_normal((n, n)) for n in ns]
    N = int(np.prod(ns))

    def multi(i):  # flat index -> (i_1, .., i_d), i_1 fastest
        out = []
        for n in ns:
            out.append(i % n)
            i //= n
        return out

    E = np.zeros((N, N))
    for i in range(N):
        ii = multi(i)
        for j in range(N):
            jj = multi(j)
            E[i, j] = sum(np.prod([(Ks[l] if l == k else Ms[l])[ii[l], jj[l]] for l in range(d)]) for k in range(d))
    np.testing.assert_allclose(assembly.kron_preconditioner_dense(Ms, Ks), E, rtol=1e-13, atol=1e-13)
    np.testing.assert_allclose(assembly.kron_preconditioner_sparse(Ms, Ks).toarray(), E, rtol=1e-13, atol=1e-13)

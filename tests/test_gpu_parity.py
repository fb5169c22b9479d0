"""GPU parity: libfdiga (C ABI, sm_100a kernels) against the CPU oracle on the same seeded inputs.

Bars (BASELINE.json north_star): fd_apply and the matvec <= 1e-12 relative l2 (FP64); GMRES iteration
counts within +-1 of the oracle at relative residual 1e-8.  fd_apply parity feeds BOTH sides the same
factors (U, W, lam) computed by the oracle (two correct setups differ by ~1e-11 through
cond(P) ~ 1e5); the library's own setup is checked separately by residuals.
"""
import json
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1705_04384_b200 as fd  # noqa: E402
from oracle import assembly, fastdiag, krylov, splines  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector, get_config, rhs  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_gmres.json")))
DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def ctx():
    c = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


# ----------------------------------------------------------------------------- FD apply

def _random_factors(ns, seed):
    rng = np.random.default_rng(seed)
    U = [rng.standard_normal((n, n)) for n in ns]
    lam = [rng.uniform(1, 100, n) for n in ns]
    return fastdiag.factors_from_eig(U, lam), rng


@pytest.mark.parametrize("ns", [(1, 1, 1), (2, 3, 5), (7, 9, 11), (33, 17, 40), (65, 65, 65), (130, 3, 129),
                                (131, 131, 131), (1, 1), (32, 32), (257, 257), (129, 300), (16, 16, 16)])
def test_fd_apply_matches_oracle_shared_factors(ctx, ns):
    f, rng = _random_factors(ns, 100 + sum(ns))
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    r = rng.standard_normal(int(np.prod(ns)))
    s = torch.empty(r.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(r), s)
    expect = fastdiag.apply(f, r)
    assert rel(host(s), expect) <= 1e-12


@pytest.mark.parametrize("n,path", [(128, None), (256, None), (512, None), (256, "dmma"), (512, "dmma")])
def test_fd_apply_cfg4_full_size(ctx, n, path):
    # BASELINE.json configs[3]: U ~ N(0,1), lam ~ U(1,100), x ~ N(0,1); W = U^{-1} from the oracle.  path None:
    # the default rule (int8-split at 256 / 512); "dmma": the IEEE FP64 DMMA products at the headline sizes
    rng, U, lam = fd_sweep_factors(n)
    f = fastdiag.factors_from_eig(U, lam)
    x = fd_sweep_vector(rng, n ** 3)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    if path:
        plan.set_path(path)
        assert plan.path()[0] == path
    s = torch.empty(n ** 3, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(x), s)
    assert rel(host(s), fastdiag.apply(f, x)) <= 1e-12
    assert plan.flops() == 12 * n ** 4


def test_fd_apply_aliasing_and_misaligned_views(ctx):
    ns = (33, 35, 37)
    f, rng = _random_factors(ns, 5)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    N = int(np.prod(ns))
    r = rng.standard_normal(N)
    buf = torch.zeros(N + 1, dtype=torch.float64, device=DEV)
    view = buf[1:]                     # 8-byte (not 16-byte) aligned device pointer
    view.copy_(gpu(r))
    fd.fd_apply(plan, view, view)      # s aliases r
    assert rel(host(view), fastdiag.apply(f, r)) <= 1e-12


def test_fd_apply_host_entry(ctx):
    ns = (20, 21, 22)
    f, rng = _random_factors(ns, 9)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    r = rng.standard_normal(int(np.prod(ns)))
    s = np.empty_like(r)
    fd.fd_apply_host(plan, r, s)
    assert rel(s, fastdiag.apply(f, r)) <= 1e-12


def test_fd_setup_from_eig_computes_inverse(ctx):
    rng, U, lam = fd_sweep_factors(96)
    plan = fd.fd_setup_from_eig(ctx, U, lam)
    for l in range(3):
        Ug, Wg, lr, li = plan.factors(l)
        assert np.linalg.norm(Wg @ U[l] - np.eye(96)) <= 1e-10
        np.testing.assert_array_equal(lr, lam[l])


@pytest.mark.parametrize("ne,p,d", [(32, 2, 2), (256, 3, 2), (64, 3, 3), (128, 5, 3), (9, 4, 3)])
def test_fd_setup_pencils_by_residuals(ctx, ne, p, d):
    # the library's own generalized eigendecomposition (cuSOLVER) on the collocation pencils
    _, M, K, _ = splines.colloc_1d(ne, p)
    plan = fd.fd_setup(ctx, [M] * d, [K] * d)
    _, _, lam_o, _ = fastdiag.setup_direction(M, K)
    for l in range(d):
        U, W, lam, lam_im = plan.factors(l)
        assert np.all(lam_im == 0) and np.all(np.diff(lam) >= 0)
        np.testing.assert_allclose(np.linalg.norm(U, axis=0), 1.0, atol=1e-13)
        assert np.linalg.norm(K @ U - M @ U @ np.diag(lam)) / (np.linalg.norm(K) * np.linalg.norm(U)) < 1e-13
        assert np.linalg.norm(W @ M @ U - np.eye(len(lam))) < 1e-10
        np.testing.assert_allclose(lam, lam_o, rtol=1e-9)
    # the apply with the library's own factors solves P s = b (exact solver)
    b = rhs(0, M.shape[0] ** d)
    s = torch.empty(b.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(b), s)
    P = assembly.kron_preconditioner_sparse([M] * d, [K] * d)
    assert np.linalg.norm(P @ host(s) - b) / np.linalg.norm(b) <= 1e-11


def test_fd_setup_rejects_complex_spectrum(ctx):
    # rotation pencil: M = I, K = [[1, -5], [5, 1]] has eigenvalues 1 +- 5i (P:434 complex case)
    K = np.array([[1.0, -5.0], [5.0, 1.0]])
    with pytest.raises(fd.FdigaError) as e:
        fd.fd_setup(ctx, [np.eye(2)] * 2, [K] * 2)
    assert e.value.status == -5


def test_fd_setup_rejects_singular_sums(ctx):
    U = [np.eye(3)] * 2
    with pytest.raises(fd.FdigaError) as e:
        fd.fd_setup_from_factors(ctx, U, U, [np.array([-1.0, 0.5, 2.0]), np.array([1.0, 3.0, 4.0])])
    assert e.value.status == -7


# ---- complex pairs in real 2x2-block form: convection-diffusion pencils (eq:convec_prec_2)

def _fd_tol(f):
    """FP64 forward error of the apply grows with prod_l cond(U_l) (the Kronecker transforms, DESIGN.md
    "Tolerances"): the north-star 1e-12 bar is kept up to prod cond = 1e4 (the Poisson pencils have
    prod cond <= 9.2^3) and scaled linearly beyond."""
    kappa = float(np.prod([np.linalg.cond(u) for u in f.U]))
    return 1e-12 * max(1.0, kappa / 1e4)


@pytest.mark.parametrize("d,wind,ne", [(2, 100.0, 6), (3, 100.0, 5), (2, 1000.0, 33), (3, 200.0, 12),
                                       (2, 10000.0, 128), (3, 1000.0, 40), (2, 25.0, 9), (3, 60.0, 7),
                                       (3, 100.0, 17)])
def test_fd_apply_complex_pairs_shared_factors(ctx, d, wind, ne):
    M, K, H = splines.galerkin_1d(ne, 2, wind)
    f = fastdiag.setup([M] * d, [K + H] * d, allow_complex=True)
    assert f.has_pairs
    plan = fd.fd_setup_from_blocks(ctx, f.U, f.W, f.lam, f.lam_im)
    b = np.random.default_rng(ne + d).standard_normal(ne ** d)
    s = torch.empty(b.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(b), s)
    assert rel(host(s), fastdiag.apply(f, b)) <= _fd_tol(f)


def test_fd_apply_complex_pairs_mixed_directions(ctx):
    # one direction all-complex, one mixed, one real: blocks of size 1, 2 and 4 side by side
    M1, K1, H1 = splines.galerkin_1d(12, 2, 200.0)
    M2, K2, H2 = splines.galerkin_1d(9, 2, 25.0)
    M3, K3, _ = splines.galerkin_1d(7, 2, 0.0)
    f = fastdiag.setup([M1, M2, M3], [K1 + H1, K2 + H2, K3], allow_complex=True)
    plan = fd.fd_setup_from_blocks(ctx, f.U, f.W, f.lam, f.lam_im)
    b = np.random.default_rng(3).standard_normal(12 * 9 * 7)
    s = torch.empty(b.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(b), s)
    assert rel(host(s), fastdiag.apply(f, b)) <= _fd_tol(f)


@pytest.mark.parametrize("d,wind,ne", [(2, 100.0, 16), (3, 100.0, 8), (2, 1000.0, 40), (2, 25.0, 9)])
def test_fd_setup_complex_pairs_by_residuals(ctx, d, wind, ne):
    # the library's own complex-pair setup: M^{-1}(K+H) U = U D with real 2x2 blocks, W M U = I, and the
    # apply solves P s = b (P materialised by Kronecker products, brute force)
    M, K, H = splines.galerkin_1d(ne, 2, wind)
    with pytest.raises(fd.FdigaError) as e:
        fd.fd_setup(ctx, [M] * d, [K + H] * d)
    assert e.value.status == -5
    plan = fd.fd_setup(ctx, [M] * d, [K + H] * d, allow_complex_pairs=True)
    for l in range(d):
        U, W, lr, li = plan.factors(l)
        assert np.any(li != 0)
        D = fastdiag.FDFactors([U], [W], [lr], [li]).D(0)
        assert np.linalg.norm((K + H) @ U - M @ U @ D) / (np.linalg.norm(K + H) * np.linalg.norm(U)) < 1e-13
        assert np.linalg.norm(W @ M @ U - np.eye(ne)) < 1e-10
        # the spectrum agrees with the oracle's QZ as a multiset a +- ib
        _, _, lo, lio = fastdiag.setup_direction(M, K + H, allow_complex=True)
        np.testing.assert_allclose(np.sort_complex(lr + 1j * li), np.sort_complex(lo + 1j * lio), rtol=1e-9)
    P = assembly.kron_preconditioner_dense([M] * d, [K + H] * d)
    b = rhs(0, ne ** d)
    s = torch.empty(b.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(b), s)
    assert np.linalg.norm(P @ host(s) - b) / np.linalg.norm(b) <= 1e-11


def test_fd_setup_from_blocks_rejects_malformed_pairs(ctx):
    U = [np.eye(3)] * 2
    bad = [np.array([1.0, 0.0, 0.0]), np.zeros(3)]           # +b without its -b partner
    with pytest.raises(fd.FdigaError) as e:
        fd.fd_setup_from_blocks(ctx, U, U, [np.array([2.0, 2.0, 5.0])] * 2, bad)
    assert e.value.status == -1


# ----------------------------------------------------------------------------- matvec / assembly

def _disc(cfg, ne=None):
    c = get_config(cfg)
    return c, assembly.Discretisation(c.d, c.p, ne or c.ne, c.geometry, c.geo_params)


@pytest.mark.parametrize("cfg,ne", [(1, None), (2, None), (3, None), (5, None), (2, 5), (3, 3), (5, 2), (5, 7),
                                    (3, 1)])
def test_matvec_matches_oracle(ctx, cfg, ne):
    c, disc = _disc(cfg, ne)
    A = fd.colloc_assemble(ctx, c.d, c.p, ne or c.ne, c.geometry, c.geo_params)
    assert A.N == disc.N
    x = np.random.default_rng(cfg * 7 + (ne or 0)).standard_normal(disc.N)
    y = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    fd.stencil_matvec(A, gpu(x), y)
    assert rel(host(y), disc.matvec(x)) <= 1e-12


def test_stored_values_match_oracle_rows(ctx):
    c, disc = _disc(3, 6)
    A = fd.colloc_assemble(ctx, c.d, c.p, 6, c.geometry, c.geo_params)
    vals = A.values()
    Aref = disc.assemble_csr()
    # reconstruct the dense matrix from the tensor-window layout via the library's windows
    dense = np.zeros((disc.N, disc.N))
    n = disc.n
    st, wd = A.windows()   # same 1D space in every direction
    off = 0
    for i3 in range(n):
        for i2 in range(n):
            for i1 in range(n):
                row = i1 + n * (i2 + n * i3)
                for a in range(wd[i3]):
                    for b in range(wd[i2]):
                        for cc in range(wd[i1]):
                            col = (st[i1] + cc) + n * ((st[i2] + b) + n * (st[i3] + a))
                            dense[row, col] = vals[off]
                            off += 1
    assert off == A.nnz
    np.testing.assert_allclose(dense, Aref.toarray(), atol=1e-12 * np.abs(vals).max())


def test_stencil_create_roundtrip(ctx):
    c, disc = _disc(5, 3)
    A = fd.colloc_assemble(ctx, c.d, c.p, 3, c.geometry, c.geo_params)
    vals = A.values()
    n = disc.n
    st, wd = A.windows()
    B = fd.stencil_create(ctx, [n] * 3, [st] * 3, [wd] * 3, vals)
    x = np.random.default_rng(1).standard_normal(disc.N)
    y1 = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    y2 = torch.empty_like(y1)
    fd.stencil_matvec(A, gpu(x), y1)
    fd.stencil_matvec(B, gpu(x), y2)
    np.testing.assert_array_equal(host(y1), host(y2))


# ----------------------------------------------------------------------------- GMRES

@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_gmres_iterations_match_oracle(ctx, cfg):
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    b = gpu(rhs(cfg, A.N))
    x = torch.empty_like(b)
    rep = fd.gmres_solve(ctx, A, P, b, x)
    ref = GOLD["configs"][str(cfg)]
    assert rep["converged"]
    assert abs(rep["iters"] - ref["iters"]) <= 1, (rep, ref)
    assert rep["rel_res_true"] <= 1e-8
    assert rep["rel_res_true"] <= 10 * max(rep["rel_res_implicit"], 1e-15) or rep["rel_res_true"] < 1e-12
    if cfg == 1:
        assert rep["iters"] == 1
    # the solution satisfies the ORACLE's operator too
    disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
    xh = host(x)
    bh = host(b)
    assert np.linalg.norm(bh - disc.matvec(xh)) / np.linalg.norm(bh) <= 2e-8


@pytest.mark.parametrize("cfg", [3, 5])
def test_gmres_profiled_breakdown(ctx, cfg):
    # gmres_opts.profile: the stages partition the device time of the (eagerly launched) solve, and the
    # solve takes exactly the decisions of the graph-launched one (same kernels, same order)
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=(cfg == 5))
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    b = gpu(rhs(cfg, A.N))
    x1 = torch.empty_like(b)
    x2 = torch.empty_like(b)
    r1 = fd.gmres_solve(ctx, A, P, b, x1)
    r2 = fd.gmres_solve(ctx, A, P, b, x2, profile=True)
    assert r2["iters"] == r1["iters"] and r2["rel_res_true"] == r1["rel_res_true"]
    np.testing.assert_array_equal(host(x1), host(x2))
    parts = [r2[k] for k in ("t_fd_ms", "t_matvec_ms", "t_orth_ms", "t_comm_ms", "t_other_ms")]
    assert all(p >= 0 for p in parts), parts
    assert r2["t_fd_ms"] > 0 and r2["t_matvec_ms"] > 0 and r2["t_orth_ms"] > 0
    assert r2["t_comm_ms"] == 0.0  # one rank, no process group
    assert abs(sum(parts) - r2["t_total_ms"]) <= 0.02 * r2["t_total_ms"] + 0.01, (parts, r2["t_total_ms"])
    # an unprofiled report carries no breakdown
    assert "t_fd_ms" not in r1
    P.close()
    A.close()


def test_gmres_small_matches_oracle_solution(ctx):
    c = get_config(2)
    ne = 16
    A = fd.colloc_assemble(ctx, 2, 3, ne, c.geometry, c.geo_params)
    disc = assembly.Discretisation(2, 3, ne, c.geometry, c.geo_params)
    f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
    P = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    bh = rhs(2, disc.N, rep=3)
    x = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    rep = fd.gmres_solve(ctx, A, P, gpu(bh), x, rtol=1e-12, history=True)
    xo, repo = krylov.gmres(disc.matvec, bh, precond=lambda v: fastdiag.apply(f, v), rtol=1e-12)
    assert abs(rep["iters"] - repo["iters"]) <= 1
    assert rel(host(x), xo) <= 1e-9
    # implicit residual histories agree step by step while well above rounding
    k = min(len(rep["history"]), len(repo["history"])) - 2
    np.testing.assert_allclose(rep["history"][:k], repo["history"][:k], rtol=1e-5)


def test_gmres_unpreconditioned_and_restart(ctx):
    c = get_config(1)
    A = fd.colloc_assemble(ctx, 2, 2, 8, 0)
    disc = assembly.Discretisation(2, 2, 8, 0)
    bh = rhs(1, disc.N)
    x = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    rep = fd.gmres_solve(ctx, A, None, gpu(bh), x, m=5, max_iters=500)
    xo, repo = krylov.gmres(disc.matvec, bh, m=5, max_iters=500)
    assert rep["converged"] and rep["restarts"] > 1
    assert abs(rep["iters"] - repo["iters"]) <= 2
    assert rel(host(x), xo) <= 1e-6


def test_gmres_not_converged_status(ctx):
    A = fd.colloc_assemble(ctx, 2, 3, 32, 1, (1.0, 2.0))
    b = gpu(rhs(2, A.N))
    x = torch.empty_like(b)
    rep = fd.gmres_solve(ctx, A, None, b, x, max_iters=10, raise_on_nonconvergence=False)
    assert rep["status"] == -8 and not rep["converged"] and rep["iters"] == 10


def test_kernel_launch_counter(ctx):
    f, rng = _random_factors((8, 8, 8), 1)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    r = gpu(rng.standard_normal(512))
    before = ctx.kernel_launches()
    fd.fd_apply(plan, r, r)
    assert ctx.kernel_launches() - before == 6


# ----------------------------------------------------------------------------- BiCGStab

@pytest.mark.parametrize("cfg", [1, 2, 3, 5])
def test_bicgstab_iterations_match_oracle(ctx, cfg):
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    b = gpu(rhs(cfg, A.N))
    x = torch.empty_like(b)
    for _ in range(2):  # the second solve replays the captured chunk graph
        rep = fd.bicgstab_solve(ctx, A, P, b, x)
        ref = GOLD["configs"][str(cfg)]
        assert rep["converged"] and not rep["breakdown"]
        assert abs(rep["iters"] - ref["bicgstab_iters"]) <= 1.0, (rep, ref)
        assert rep["iters"] % 1 == (0.5 if rep["half"] else 0.0)
        assert rep["rel_res_true"] <= 2e-8
    if cfg == 1:
        assert rep["iters"] == 0.5  # FD is exact on the identity map
    disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
    bh = host(b)
    assert np.linalg.norm(bh - disc.matvec(host(x))) / np.linalg.norm(bh) <= 2e-8


def test_bicgstab_small_matches_oracle_history(ctx):
    c = get_config(2)
    ne = 16
    A = fd.colloc_assemble(ctx, 2, 3, ne, c.geometry, c.geo_params)
    disc = assembly.Discretisation(2, 3, ne, c.geometry, c.geo_params)
    f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
    P = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    bh = rhs(2, disc.N, rep=5)
    x = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    rep = fd.bicgstab_solve(ctx, A, P, gpu(bh), x, rtol=1e-11, history=True)
    xo, repo = krylov.bicgstab(disc.matvec, bh, precond=lambda v: fastdiag.apply(f, v), rtol=1e-11)
    assert abs(rep["iters"] - repo["iters"]) <= 1.0
    assert rel(host(x), xo) <= 1e-9
    k = min(len(rep["history"]), len(repo["history"])) - 2
    np.testing.assert_allclose(rep["history"][:k], repo["history"][:k], rtol=1e-5)


def test_bicgstab_unpreconditioned_and_status(ctx):
    A = fd.colloc_assemble(ctx, 2, 2, 8, 0)
    disc = assembly.Discretisation(2, 2, 8, 0)
    bh = rhs(1, disc.N)
    x = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    rep = fd.bicgstab_solve(ctx, A, None, gpu(bh), x, rtol=1e-10, max_iters=500)
    xo, repo = krylov.bicgstab(disc.matvec, bh, rtol=1e-10, max_iters=500)
    assert rep["converged"] and abs(rep["iters"] - repo["iters"]) <= 2
    assert rel(host(x), xo) <= 1e-6
    A2 = fd.colloc_assemble(ctx, 2, 3, 32, 1, (1.0, 2.0))
    b2 = gpu(rhs(2, A2.N))
    x2 = torch.empty_like(b2)
    rep = fd.bicgstab_solve(ctx, A2, None, b2, x2, max_iters=3, raise_on_failure=False)
    assert rep["status"] == -8 and not rep["converged"] and rep["iters"] == 3.0


# ----------------------------------------------------------------------------- matrix-free operator (NEXT-1)

@pytest.mark.parametrize("cfg,ne", [(3, None), (5, None), (3, 1), (3, 3), (5, 2), (5, 7), (5, 13), (3, 17)])
def test_matrix_free_matvec_matches_oracle(ctx, cfg, ne):
    c, disc = _disc(cfg, ne)
    A = fd.colloc_assemble(ctx, c.d, c.p, ne or c.ne, c.geometry, c.geo_params, matrix_free=True)
    assert A.N == disc.N
    x = np.random.default_rng(cfg * 11 + (ne or 0)).standard_normal(disc.N)
    y = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    fd.stencil_matvec(A, gpu(x), y)
    assert rel(host(y), disc.matvec(x)) <= 1e-12
    with pytest.raises(fd.FdigaError):
        A.values()


def test_matrix_free_identity_map_is_kronecker(ctx):
    # identity map: A_C = K (x) M (x) M + M (x) K (x) M + M (x) M (x) K (eq:colloc3D)
    _, M, K, _ = splines.colloc_1d(9, 4)
    n = M.shape[0]
    A = fd.colloc_assemble(ctx, 3, 4, 9, 0, matrix_free=True)
    P = assembly.kron_preconditioner_sparse([M] * 3, [K] * 3)
    x = np.random.default_rng(4).standard_normal(n ** 3)
    y = torch.empty(n ** 3, dtype=torch.float64, device=DEV)
    fd.stencil_matvec(A, gpu(x), y)
    assert rel(host(y), P @ x) <= 1e-12


@pytest.mark.parametrize("cfg", [3, 5])
def test_matrix_free_gmres_and_bicgstab(ctx, cfg):
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=True)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    b = gpu(rhs(cfg, A.N))
    x = torch.empty_like(b)
    ref = GOLD["configs"][str(cfg)]
    rep = fd.gmres_solve(ctx, A, P, b, x)
    assert rep["converged"] and abs(rep["iters"] - ref["iters"]) <= 1 and rep["rel_res_true"] <= 1e-8
    rep = fd.bicgstab_solve(ctx, A, P, b, x)
    assert rep["converged"] and abs(rep["iters"] - ref["bicgstab_iters"]) <= 1.0


@pytest.mark.parametrize("cfg", [2, 5])
def test_gmres_orthogonalisation_variants_agree(ctx, cfg):
    # CGS + DGKS, CGS2 and DCGS2 (default) take the same number of steps (SURVEY.md §0.8:
    # orthogonalisation-independent counts) and reach the same solution
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=(c.d == 3))
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    b = gpu(rhs(cfg, A.N))
    x1, x2 = torch.empty_like(b), torch.empty_like(b)
    x3 = torch.empty_like(b)
    r1 = fd.gmres_solve(ctx, A, P, b, x1, orth=fd.ORTH_CGS_DGKS, history=True)
    r2 = fd.gmres_solve(ctx, A, P, b, x2, orth=fd.ORTH_CGS2, history=True)
    r3 = fd.gmres_solve(ctx, A, P, b, x3, orth=fd.ORTH_DCGS2, history=True)
    assert r1["iters"] == r2["iters"] == r3["iters"] == GOLD["configs"][str(cfg)]["iters"]
    assert r2["reorth"] == r2["iters"] and 0 <= r1["reorth"] <= r1["iters"]
    assert rel(host(x1), host(x2)) <= 1e-7 and rel(host(x3), host(x2)) <= 1e-7
    assert r3["rel_res_true"] <= 1e-8
    # delayed re-orthogonalisation builds the same Hessenberg columns: the implicit residuals agree
    np.testing.assert_allclose(r3["history"], r2["history"], rtol=1e-6)


@pytest.mark.parametrize("m", [1, 2, 5, 30])
def test_gmres_dcgs2_matches_oracle(ctx, m):
    # DCGS2 across restart lengths (m = 1: one step and the closing pass per cycle), preconditioned and
    # restarted: the oracle's GMRES(m) iteration count and solution
    A = fd.colloc_assemble(ctx, 2, 3, 16, 1, (1.0, 2.0))
    disc = assembly.Discretisation(2, 3, 16, 1, (1.0, 2.0))
    f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
    P = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    bh = rhs(2, disc.N, rep=5)
    x = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    rep = fd.gmres_solve(ctx, A, P, gpu(bh), x, m=m, max_iters=3000, rtol=1e-10, orth=fd.ORTH_DCGS2)
    xo, repo = krylov.gmres(disc.matvec, bh, precond=lambda v: fastdiag.apply(f, v), m=m, max_iters=3000,
                            rtol=1e-10)
    assert rep["converged"] and repo["converged"]
    assert abs(rep["iters"] - repo["iters"]) <= max(2, repo["iters"] // 50), (rep, repo)
    assert rel(host(x), xo) <= 1e-6


# ----------------------------------------------------------------------------- NEXT-4: convection-diffusion

@pytest.mark.parametrize("d,geom,params,wind,wp,ne,mf", [
    (3, 3, (1.0, 2.0, 1.0), 2, (3000.0,), 7, False), (3, 3, (1.0, 2.0, 1.0), 2, (3000.0,), 7, True),
    (3, 2, (0.1,), 1, (1.0, -2.0, 4.0), 6, False), (3, 2, (0.1,), 1, (1.0, -2.0, 4.0), 9, True),
    (3, 0, (), 2, (5.0,), 5, True), (2, 1, (1.0, 2.0), 2, (7.0,), 9, False),
    (3, 3, (1.0, 2.0, 1.0), 2, (10.0,), None, True)])
def test_convection_operator_matches_oracle(ctx, d, geom, params, wind, wp, ne, mf):
    p = 5 if d == 3 else 3
    ne = ne or 128
    disc = assembly.Discretisation(d, p, ne, geom, params, wind=wind, wind_params=wp)
    A = fd.colloc_assemble(ctx, d, p, ne, geom, params, matrix_free=mf, wind=wind, wind_params=wp)
    x = np.random.default_rng(ne + wind).standard_normal(disc.N)
    y = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    fd.stencil_matvec(A, gpu(x), y)
    assert rel(host(y), disc.matvec(x)) <= 1e-12


def test_convection_factor_matches_oracle():
    wt = np.linspace(-3.0, 5.0, 11)
    np.testing.assert_allclose(fd.colloc_1d_convection(3, 10, wt), splines.colloc_1d_convection(10, 3, wt),
                               rtol=1e-13, atol=1e-13)


@pytest.mark.parametrize("cfg", [6, 7])
def test_convection_gmres_wind_aware_fd(ctx, cfg):
    # eq:convec_prec_2 (collocation analogue): K_2 + H_2 with w~_2 = 2 omega / pi; complex pairs at cfg 6
    c = get_config(cfg)
    ref = GOLD["next4"][str(cfg)]
    A = fd.colloc_assemble(ctx, 3, c.p, c.ne, c.geometry, c.geo_params, matrix_free=True, wind=c.wind,
                           wind_params=c.wind_params)
    M, K = fd.colloc_1d_factors(c.p, c.ne)
    H2 = fd.colloc_1d_convection(c.p, c.ne, 2 * c.wind_params[0] / np.pi)
    Pw = fd.fd_setup(ctx, [M] * 3, [K, K + H2, K], allow_complex_pairs=True, cond_max=1e30)
    assert np.any(Pw.factors(1)[3] != 0) == ref["has_complex_pairs"]
    b = gpu(rhs(cfg, A.N))
    x = torch.empty_like(b)
    rep = fd.gmres_solve(ctx, A, Pw, b, x, max_iters=300)
    assert rep["converged"] and abs(rep["iters"] - ref["iters_wind_fd"]) <= 1, (rep, ref)
    P0 = fd.fd_setup(ctx, [M] * 3, [K] * 3)
    rep0 = fd.gmres_solve(ctx, A, P0, b, x, max_iters=300, raise_on_nonconvergence=False)
    if ref["converged_plain_fd"]:
        assert abs(rep0["iters"] - ref["iters_plain_fd"]) <= 1
    else:
        assert rep0["status"] == -8 and rep0["iters"] == 300


# ----------------------------------------------------------------------------- NEXT-3: weighted quadrature

@pytest.mark.parametrize("d,p,ne,geom,params", [(2, 2, 7, 1, (1.0, 2.0)), (2, 3, 9, 1, (1.0, 2.0)),
                                                (2, 4, 8, 1, (1.0, 2.0)), (2, 5, 11, 1, (1.0, 2.0)),
                                                (3, 2, 5, 3, (1.0, 2.0, 1.0)), (3, 3, 6, 2, (0.1,)),
                                                (3, 4, 5, 0, ()), (2, 3, 1, 1, (1.0, 2.0))])
def test_wq_operator_matches_oracle(ctx, d, p, ne, geom, params):
    from oracle import quadrature
    if ne + p - 2 < 1:
        pytest.skip("empty space")
    disc = quadrature.WQDiscretisation(d, p, ne, geom, params)
    Ao = disc.assemble_wq()
    A = fd.wq_assemble(ctx, d, p, ne, geom, params)
    assert A.nnz >= Ao.nnz
    x = np.random.default_rng(d * 10 + p + ne).standard_normal(disc.N)
    y = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    fd.stencil_matvec(A, gpu(x), y)
    assert rel(host(y), Ao @ x) <= 1e-12


@pytest.mark.parametrize("cfg", [8, 9])
def test_wq_solvers_match_oracle_counts(ctx, cfg):
    c = get_config(cfg)
    ref = GOLD["wq"][str(cfg)]
    A = fd.wq_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
    M, K = fd.galerkin_1d_factors(c.p, c.ne)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    for l in range(c.d):   # symmetric positive definite pencil: real, positive spectrum (V = U)
        U, W, lam, lam_im = P.factors(l)
        assert np.all(lam_im == 0) and np.all(lam > 0)
    b = gpu(rhs(cfg, A.N))
    x = torch.empty_like(b)
    rep = fd.gmres_solve(ctx, A, P, b, x)
    assert rep["converged"] and abs(rep["iters"] - ref["iters"]) <= 1
    rb = fd.bicgstab_solve(ctx, A, P, b, x)
    assert rb["converged"] and abs(rb["iters"] - ref["bicgstab_iters"]) <= 1.0


def test_fd_apply_host_async_matches_sync(ctx):
    ns = (30, 31, 32)
    f, rng = _random_factors(ns, 21)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    N = int(np.prod(ns))
    ins = [torch.from_numpy(rng.standard_normal(N)).pin_memory() for _ in range(5)]
    outs = [torch.empty(N, dtype=torch.float64).pin_memory() for _ in range(5)]
    for a, b in zip(ins, outs):
        fd.fd_apply_host_async(plan, a.numpy(), b.numpy())
    fd.fd_host_sync(plan)
    for a, b in zip(ins, outs):
        assert rel(b.numpy(), fastdiag.apply(f, a.numpy())) <= 1e-12


# ----------------------------------------------------------------------------- degenerate and edge cases

def _small_system(ctx):
    c = get_config(2)
    A = fd.colloc_assemble(ctx, 2, 3, 12, c.geometry, c.geo_params)
    M, K = fd.colloc_1d_factors(3, 12)
    P = fd.fd_setup(ctx, [M] * 2, [K] * 2)
    return A, P


def test_solvers_zero_rhs(ctx):
    A, P = _small_system(ctx)
    b = torch.zeros(A.N, dtype=torch.float64, device=DEV)
    x = torch.full_like(b, 7.0)
    rep = fd.gmres_solve(ctx, A, P, b, x)
    assert rep["converged"] and rep["iters"] == 0 and float(x.abs().max()) == 0.0
    x.fill_(7.0)
    rep = fd.bicgstab_solve(ctx, A, P, b, x)
    assert rep["converged"] and rep["iters"] == 0.0 and float(x.abs().max()) == 0.0


def test_gmres_initial_guess_is_solution(ctx):
    A, P = _small_system(ctx)
    b = gpu(rhs(2, A.N, rep=9))
    x = torch.empty_like(b)
    fd.gmres_solve(ctx, A, P, b, x, rtol=1e-12)
    rep = fd.gmres_solve(ctx, A, P, b, x, rtol=1e-8, use_x0=True)
    assert rep["converged"] and rep["iters"] == 0
    rep = fd.bicgstab_solve(ctx, A, P, b, x, rtol=1e-8, use_x0=True)
    assert rep["converged"] and rep["iters"] == 0.0


def test_gmres_restart_length_one_matches_oracle(ctx):
    c = get_config(2)
    A, P = _small_system(ctx)
    disc = assembly.Discretisation(2, 3, 12, c.geometry, c.geo_params)
    f = fastdiag.setup([disc.M] * 2, [disc.K] * 2)
    bh = rhs(2, disc.N, rep=4)
    x = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    P2 = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    rep = fd.gmres_solve(ctx, A, P2, gpu(bh), x, m=1, max_iters=3000)
    xo, repo = krylov.gmres(disc.matvec, bh, precond=lambda v: fastdiag.apply(f, v), m=1, max_iters=3000)
    assert rep["converged"] and repo["converged"]
    assert abs(rep["iters"] - repo["iters"]) <= max(2, repo["iters"] // 20)
    assert rep["restarts"] == rep["iters"]  # GMRES(1): one step per cycle


def test_solvers_report_breakdown_on_nan(ctx):
    A, P = _small_system(ctx)
    bh = rhs(2, A.N)
    bh[5] = np.nan
    b = gpu(bh)
    x = torch.empty_like(b)
    rep = fd.gmres_solve(ctx, A, P, b, x, raise_on_nonconvergence=False)
    assert rep["status"] == -9 and not rep["converged"]
    rep = fd.bicgstab_solve(ctx, A, P, b, x, raise_on_failure=False)
    assert rep["status"] == -9 and rep["breakdown"]


def test_api_argument_errors(ctx):
    A, P = _small_system(ctx)
    x = torch.zeros(A.N, dtype=torch.float64, device=DEV)
    with pytest.raises(fd.FdigaError) as e:
        fd.stencil_matvec(A, x, x)          # aliasing is rejected by the library
    assert e.value.status == -1
    with pytest.raises(ValueError):
        fd.fd_apply(P, x[:-1], x[:-1])      # wrong length (binding check)
    with pytest.raises(TypeError):
        fd.fd_apply(P, x.float(), x.float())
    with pytest.raises(fd.FdigaError):
        fd.gmres_solve(ctx, A, P, x, torch.zeros_like(x), m=40)   # m > 31


def test_fd_apply_large_2d_ragged(ctx):
    # a large, ragged 2D apply (n = 3001 and 2049: 6.1M DOF) against the oracle's mode products
    ns = (3001, 2049)
    f, rng = _random_factors(ns, 77)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    r = rng.standard_normal(int(np.prod(ns)))
    s = torch.empty(r.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(r), s)
    assert rel(host(s), fastdiag.apply(f, r)) <= 1e-12


def test_nvtx_stage_ranges_leave_the_solve_unchanged():
    """FDIGA_NVTX=1 (NVTX ranges per API call and per solve stage, read once per process) must not change
    results: the exactly preconditioned cfg1 solve still takes 1 iteration, profiled and graph-launched."""
    import subprocess
    import sys
    code = (
        "import torch, paper_1705_04384_b200 as fd\n"
        "from synth import get_config, rhs\n"
        "ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)\n"
        "c = get_config(1)\n"
        "A = fd.colloc_assemble(ctx, 2, c.p, c.ne, c.geometry)\n"
        "M, K = fd.colloc_1d_factors(c.p, c.ne)\n"
        "P = fd.fd_setup(ctx, [M, M], [K, K])\n"
        "b = torch.from_numpy(rhs(1, A.N)).cuda(); x = torch.empty_like(b)\n"
        "for prof in (False, True):\n"
        "    rep = fd.gmres_solve(ctx, A, P, b, x, profile=prof)\n"
        "    assert rep['converged'] and rep['iters'] == 1, rep\n"
        "rep = fd.bicgstab_solve(ctx, A, P, b, x)\n"
        "assert rep['converged'], rep\n"
        "print('nvtx ok')\n"
    )
    env = dict(os.environ, FDIGA_NVTX="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], env=env, cwd=root, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0 and "nvtx ok" in out.stdout, out.stderr[-2000:]

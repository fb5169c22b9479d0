"""GPU parity of the int8-split tensor-core FD path (oz.cu: exact int8 digit splitting on
tcgen05.mma.kind::i8) against the CPU oracle.

The path is forced with FDIGA_FD_OZ=1 (read when a plan is set up) so that ragged, tiny, Poisson and long
(K > 256: streamed factor digits) shapes go through it; the default rule (3D, real spectra,
192 <= n_l <= 512) is checked separately; the sharded
variants are in test_gpu_sharded.py.  Bar: the
north_star's 1e-12 relative l2 for fd_apply, GMRES counts within +-1 of the oracle.
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
from oracle import fastdiag, splines  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector, get_config, rhs  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_gmres.json")))
DEV = torch.device("cuda:0")


def rel(a, b):
    sc = float(np.max(np.abs(b))) or 1.0  # scaled: the 2^540 rows would overflow the squared norms
    return float(np.linalg.norm((a - b) / sc) / np.linalg.norm(b / sc))


@pytest.fixture(scope="module")
def ctx():
    c = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


@pytest.fixture
def forced(monkeypatch):
    monkeypatch.setenv("FDIGA_FD_OZ", "1")


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x)).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def _random_factors(ns, seed):
    rng = np.random.default_rng(seed)
    U = [rng.standard_normal((n, n)) for n in ns]
    lam = [rng.uniform(1, 100, n) for n in ns]
    return fastdiag.factors_from_eig(U, lam), rng


@pytest.mark.parametrize("ns", [(1, 1, 1), (2, 3, 5), (7, 9, 11), (16, 16, 16), (33, 17, 40), (65, 65, 65),
                                (130, 3, 129), (131, 131, 131), (200, 256, 192), (300, 40, 36), (20, 300, 24),
                                (24, 20, 400)])
def test_int8_fd_apply_matches_oracle(ctx, forced, ns):
    f, rng = _random_factors(ns, 300 + sum(ns))
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    assert plan.path()[0] == "int8_split"
    r = rng.standard_normal(int(np.prod(ns)))
    s = torch.empty(r.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(r), s)
    assert rel(host(s), fastdiag.apply(f, r)) <= 1e-12


def test_int8_cfg4_n256_is_the_default_path(ctx):
    # BASELINE.json configs[3] at n = 256 takes the int8 path without any override
    rng, U, lam = fd_sweep_factors(256)
    f = fastdiag.factors_from_eig(U, lam)
    x = fd_sweep_vector(rng, 256 ** 3)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    path, ops = plan.path()
    assert path == "int8_split"
    assert ops == 6 * 2 * 34 * 65536 * 256 * 256  # six products, 34 digit pairs each, unpadded shapes
    s = torch.empty(x.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(x), s)
    assert rel(host(s), fastdiag.apply(f, x)) <= 1e-12


@pytest.mark.parametrize("ns,expect", [((128, 128, 128), "dmma"), ((131, 131, 131), "dmma"),
                                       ((256, 256, 256), "int8_split"), ((512, 512, 512), "int8_split"),
                                       ((256, 256, 512), "int8_split"), ((513, 256, 256), "dmma"),
                                       ((256, 256), "dmma")])
def test_int8_default_rule(ctx, ns, expect):
    U = [np.eye(n) for n in ns]
    lam = [np.linspace(1.0, 2.0, n) for n in ns]
    plan = fd.fd_setup_from_eig(ctx, U, lam)
    assert plan.path()[0] == expect


def test_int8_override_off(ctx, monkeypatch):
    monkeypatch.setenv("FDIGA_FD_OZ", "0")
    plan = fd.fd_setup_from_eig(ctx, [np.eye(256)] * 3, [np.linspace(1, 2, 256)] * 3)
    assert plan.path() == ("dmma", 0.0)


@pytest.mark.parametrize("sc", [300, 540])
def test_int8_zero_and_scaled_rows(ctx, forced, sc):
    # zero rows (exponent 0, all digits 0) and rows 2^+-sc apart: the per-row exponents keep every row's
    # relative accuracy (a shared scale would flush the small rows).  Mode-3 fibres span both scales; at
    # sc = 540 the small values underflow when scaled by the fibre's exponent, and a negative one must still
    # floor to -1 (the splits round the scaling down)
    ns = (48, 40, 36)
    f, rng = _random_factors(ns, 7)
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    s = torch.empty(int(np.prod(ns)), dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, torch.zeros_like(s), s)
    assert not host(s).any()
    r = rng.standard_normal(ns[::-1])
    r[::2] *= 2.0 ** sc
    r[1::2] *= 2.0 ** -sc
    r = r.ravel()
    fd.fd_apply(plan, gpu(r), s)
    expect = fastdiag.apply(f, r)
    got = host(s).reshape(ns[::-1])
    ex = expect.reshape(ns[::-1])
    # the big planes dominate the global norm: check the small planes on their own too
    assert rel(got[::2].ravel(), ex[::2].ravel()) <= 1e-12
    small = fastdiag.apply(f, np.where(np.arange(ns[2])[:, None, None] % 2 == 1, r.reshape(ns[::-1]), 0).ravel())
    s2 = torch.empty_like(s)
    fd.fd_apply(plan, gpu(np.where(np.arange(ns[2])[:, None, None] % 2 == 1, r.reshape(ns[::-1]), 0).ravel()), s2)
    assert rel(host(s2), small) <= 1e-12


@pytest.mark.parametrize("cfg", [3])
def test_int8_gmres_counts(ctx, forced, cfg):
    # Poisson collocation pencils (real spectra) through the int8 FD inside GMRES(30): same iteration count
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
    M, K = fd.colloc_1d_factors(c.p, c.ne)
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    assert P.path()[0] == "int8_split"
    b = gpu(rhs(cfg, A.N))
    x = torch.empty_like(b)
    rep = fd.gmres_solve(ctx, A, P, b, x)
    ref = GOLD["configs"][str(cfg)]
    assert rep["converged"]
    assert abs(rep["iters"] - ref["iters"]) <= 1, (rep, ref)
    assert rep["rel_res_true"] <= 1e-8


def test_int8_poisson_pencils_match_oracle(ctx, forced):
    # the library's own setup from the 1D collocation pencils, applied on the int8 path, against
    # the oracle's P^{-1} b with the same pencils; the setups differ by ~cond(P) eps, hence the looser bar
    ne, p = 40, 3
    M, K = fd.colloc_1d_factors(p, ne)
    P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
    assert P.path()[0] == "int8_split"
    _, Mo, Ko, _ = splines.colloc_1d(ne, p)
    f = fastdiag.setup([Mo] * 3, [Ko] * 3)
    n = M.shape[0]
    rng = np.random.default_rng(11)
    b = rng.uniform(-1, 1, n ** 3)
    s = torch.empty(n ** 3, dtype=torch.float64, device=DEV)
    fd.fd_apply(P, gpu(b), s)
    assert rel(host(s), fastdiag.apply(f, b)) <= 1e-10


def test_fd_apply_timed_reports_every_kernel(ctx, monkeypatch):
    # fd_apply_timed: one event-timed step per launched kernel, kinds by path; same result as fd_apply
    ns = (24, 20, 16)
    f, rng = _random_factors(ns, 5)
    r = gpu(rng.standard_normal(int(np.prod(ns))))
    for force, kinds in (("1", ["split", "int8_gemm"] * 6), ("0", ["dmma"] * 6)):
        monkeypatch.setenv("FDIGA_FD_OZ", force)
        plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
        s1 = torch.empty_like(r)
        s2 = torch.empty_like(r)
        steps = fd.fd_apply_timed(plan, r, s1)
        fd.fd_apply(plan, r, s2)
        assert [k for k, _ in steps] == kinds
        assert all(ms > 0 for _, ms in steps)
        assert torch.equal(s1, s2)
        plan.close()

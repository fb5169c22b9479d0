"""Elementwise accuracy of fd_apply on both mode-product paths against the oracle.

  dmma        IEEE FP64 dot products: |s_gpu - s_oracle| <= B_fp64(library order) + B_fp64(oracle order)
  int8_split  the path's accuracy contract: <= B_int8 + B_fp64(oracle order)

with the a-priori bounds of tests/fd_bounds.py (pinned against exact rational arithmetic in
test_int8_split_scheme.py), checked element by element on the headline workload (BASELINE.json configs[3] at
n = 256), a ragged shape and a real cfg5 Krylov vector; and the guard (oz.cuh): fibres with a dynamic range
beyond 2^24 (2^+-30 inside one fibre, a spike against zero factor entries), NaN/Inf and out-of-range
exponents are computed as IEEE FP64 dot products, so there the int8 path meets the plain FP64 bound.
"""
import numpy as np
import pytest

from tests import fd_bounds as fb

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1705_04384_b200 as fd  # noqa: E402
from oracle import fastdiag  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector, get_config, rhs  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx():
    c = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


def gpu(x):
    return torch.from_numpy(np.ascontiguousarray(x).ravel()).to(DEV)


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def run(plan, x, path):
    plan.set_path(path)
    assert plan.path()[0] == path
    s = torch.empty(x.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, gpu(x), s)
    return host(s).reshape(x.shape)


def check_bound(f, x, got, path, ratio_max=1.0):
    """Elementwise |got - oracle| <= B_path + B_oracle; returns the worst ratio."""
    shape = x.shape
    expect = fastdiag.apply(f, x.ravel()).reshape(shape)
    Lam = fb.lam_grid(f.lam)
    _, Bp = fb.apply_bound(f.W, f.U, Lam, x, "int8" if path == "int8_split" else "fp64")
    _, Bo = fb.apply_bound(f.W, f.U, Lam, x, "fp64", bwd=(0, 1, 2))
    err = np.abs(got - expect)
    ratio = float(np.max(err / (Bp + Bo)))
    assert ratio <= ratio_max, (path, ratio)
    return ratio


@pytest.mark.parametrize("path", ["dmma", "int8_split"])
@pytest.mark.parametrize("ns", [(256, 256, 256), (200, 256, 72)])
def test_elementwise_bound_cfg4(ctx, ns, path):
    # the headline workload (BASELINE.json configs[3], n = 256) and a ragged shape
    rng, U, lam = fd_sweep_factors(ns)
    f = fastdiag.factors_from_eig(U, lam)
    x = fd_sweep_vector(rng, int(np.prod(ns))).reshape(ns[::-1])
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    got = run(plan, x, path)
    r = check_bound(f, x, got, path)
    # and far from vacuous: the measured error sits well below the a-priori bound
    assert r < 0.05, r
    plan.close()


@pytest.mark.parametrize("path", ["dmma", "int8_split"])
def test_elementwise_bound_real_cfg5_krylov_vector(ctx, path):
    # a genuine Krylov vector of the cfg5 solve (BASELINE.json configs[4]): v = A P^-1 b / ||.||, the direction
    # GMRES's first Arnoldi step produces, through the library's own operator and preconditioner
    c = get_config(5)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=True)
    M, K = fd.colloc_1d_factors(c.p, c.ne)
    P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
    b = gpu(rhs(5, A.N))
    z = torch.empty_like(b)
    v = torch.empty_like(b)
    fd.fd_apply(P, b, z)
    fd.stencil_matvec(A, z, v)
    v /= torch.linalg.norm(v)
    n = A.n[0]
    x = host(v).reshape(n, n, n)
    Us, Ws, lams = [], [], []
    for l in range(3):
        U_, W_, lr, _ = P.factors(l)
        Us.append(U_)
        Ws.append(W_)
        lams.append(lr)
    f = fastdiag.FDFactors(Us, Ws, lams)
    got = run(P, x, path)
    r = check_bound(f, x, got, path)
    assert r < 0.05, r
    P.close()
    A.close()


def _single_axis_problem(l, A_vec, others=(24, 20), seed=0, zero_col=False):
    """Factors random along axis l (length A_vec.size), identity on the other two axes with eigenvalue 0
    there (Lambda = lam_l > 0); x = A along axis l times benign U(1, 2) values across it.  Only the fibres
    along axis l carry A's dynamic range."""
    rng = np.random.default_rng(seed)
    n_l = A_vec.size
    ns = list(others)
    ns.insert(l, n_l)
    Us, Ws, lams = [], [], []
    for k, n in enumerate(ns):
        if k == l:
            Uk = rng.standard_normal((n, n))
            Wk = np.linalg.inv(Uk)
            if zero_col:   # factor rows that are zero against the fibres' large entry (index 0)
                Uk[::2, 0] = 0.0
                Wk[::2, 0] = 0.0
            Us.append(Uk)
            Ws.append(Wk)
            lams.append(rng.uniform(1, 100, n))
        else:
            Us.append(np.eye(n))
            Ws.append(np.eye(n))
            lams.append(np.zeros(n))
    shape = ns[::-1]
    B = rng.uniform(1, 2, shape)
    bshape = [1, 1, 1]
    bshape[2 - l] = n_l
    x = B * A_vec.reshape(bshape)
    return fastdiag.FDFactors(Us, Ws, lams), x


ADVERSARIAL = {
    "pm30": lambda rng, n: rng.standard_normal(n) * 2.0 ** rng.choice([-30, 30], n),
    "spike_vs_zero": lambda rng, n: np.r_[1.0, 1e-12 * rng.standard_normal(n - 1)],
}


@pytest.mark.parametrize("kind", sorted(ADVERSARIAL))
@pytest.mark.parametrize("l", [0, 1, 2])
@pytest.mark.parametrize("nl", [256, 320])  # 320: the streamed-factor GEMM (contractions > 256 in one launch)
def test_guard_wide_fibres_meet_the_fp64_bound(ctx, l, kind, nl):
    # intra-fibre dynamic range along each contracted axis: the guard sends those fibres to IEEE FP64 dot
    # products, so the int8 path meets the plain FP64 bound (B_fp64 of the library order) -- without the guard
    # the spike row's error is ~1e-5 relative (test_int8_split_scheme.py)
    rng = np.random.default_rng(10 + l)
    f, x = _single_axis_problem(l, ADVERSARIAL[kind](rng, nl), seed=l, zero_col=(kind == "spike_vs_zero"))
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    got = run(plan, x, "int8_split")
    check_bound(f, x, got, "dmma")
    plan.close()


def test_guard_nonfinite_inputs_propagate_like_fp64(ctx):
    rng = np.random.default_rng(3)
    f, x = _single_axis_problem(0, rng.standard_normal(200), seed=3)
    x = x.copy()
    x[5, 7, 11] = np.nan
    x[9, 2, 100] = np.inf
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    a = run(plan, x, "dmma")
    b = run(plan, x, "int8_split")
    assert np.array_equal(np.isnan(a), np.isnan(b))
    assert np.array_equal(np.isposinf(a), np.isposinf(b)) and np.array_equal(np.isneginf(a), np.isneginf(b))
    # IEEE: every mode product is a dense contraction (0 * NaN = NaN, 0 * Inf = NaN), so one non-finite entry
    # reaches every output; the int8 path must not turn any of them into finite values
    fin = np.isfinite(a)
    assert not fin.any()
    assert np.array_equal(np.isfinite(b), fin)
    plan.close()


def test_guard_exponents_out_of_digit_range(ctx):
    # planes at 2^-1000 (below OZ_EMIN: the digit scaling would leave the double range) and 2^+1000 next to
    # ordinary planes: mode-3 fibres span ~2000 binades -> FP64; the tiny planes alone stay accurate too
    rng = np.random.default_rng(4)
    ns = (40, 36, 32)
    U = [rng.standard_normal((n, n)) for n in ns]
    f = fastdiag.factors_from_eig(U, [rng.uniform(1, 100, n) for n in ns])
    x = rng.standard_normal(ns[::-1])
    x[::3] *= 2.0 ** -1000
    x[1::3] *= 2.0 ** 1000
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    got = run(plan, x, "int8_split")
    check_bound(f, x, got, "int8_split")
    tiny = np.where(np.arange(ns[2])[:, None, None] % 3 == 0, x, 0.0)
    got_t = run(plan, tiny, "int8_split")
    exp_t = fastdiag.apply(f, tiny.ravel()).reshape(tiny.shape)
    assert np.linalg.norm((got_t - exp_t).ravel() * 2.0 ** 1000) <= 1e-12 * np.linalg.norm(exp_t.ravel() * 2.0 ** 1000)
    plan.close()


def test_int8_offset_output_view(ctx):
    # an 8-byte (not 16-byte) aligned output on the int8 path: the mode-1 epilogue must not use 16-byte stores
    ns = (192, 10, 6)
    rng = np.random.default_rng(8)
    U = [rng.standard_normal((n, n)) for n in ns]
    f = fastdiag.factors_from_eig(U, [rng.uniform(1, 100, n) for n in ns])
    plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    plan.set_path("int8_split")
    N = int(np.prod(ns))
    r = rng.standard_normal(N)
    buf = torch.zeros(N + 1, dtype=torch.float64, device=DEV)
    out = buf[1:]
    fd.fd_apply(plan, gpu(r), out)
    expect = fastdiag.apply(f, r)
    assert np.linalg.norm(host(out) - expect) <= 1e-12 * np.linalg.norm(expect)
    plan.close()


def test_set_path_rules(ctx):
    rng = np.random.default_rng(1)
    U2 = [np.eye(8), np.eye(9)]
    p2 = fd.fd_setup_from_eig(ctx, U2, [np.linspace(1, 2, 8), np.linspace(1, 2, 9)])
    with pytest.raises(fd.FdigaError):
        p2.set_path("int8_split")          # 2D: not supported, plan unchanged
    assert p2.path()[0] == "dmma"
    p2.close()
    U = [rng.standard_normal((n, n)) for n in (20, 21, 22)]
    f = fastdiag.factors_from_eig(U, [rng.uniform(1, 100, n) for n in (20, 21, 22)])
    p3 = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    assert p3.path()[0] == "dmma"         # default rule: n_l < 192
    x = rng.standard_normal(20 * 21 * 22)
    a = run(p3, x.reshape(22, 21, 20), "int8_split")
    b = run(p3, x.reshape(22, 21, 20), "dmma")
    assert np.linalg.norm(a - b) <= 1e-12 * np.linalg.norm(b)
    p3.close()

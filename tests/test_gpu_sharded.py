"""GPU parity of the slab-sharded path on ONE device through the loopback transport.

nranks contexts share one B200, each driven by its own host thread and stream; the library's
collectives move the slabs / transpose chunks / halo planes between them device-to-device (no kernel
waits on another rank).  Every rank runs exactly the kernels and exchange schedule of the NCCL path,
so the sharded FD apply (local modes 1..d-1, slab -> chunk transpose, mode-d sandwich, transpose
back), the halo-exchanging matvec and the all-reducing GMRES are checked against the CPU oracle
with the single-GPU bars: <= 1e-12 relative l2, GMRES iterations +-1.
"""
import json
import os
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1705_04384_b200 as fd  # noqa: E402
from oracle import assembly, fastdiag, splines  # noqa: E402
from synth import get_config, rhs  # noqa: E402

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "oracle_gmres.json")))
DEV = torch.device("cuda:0")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def run_ranks(nranks, fn, timeout=300):
    """Run fn(ctx, rank) on nranks loopback contexts (one thread + stream each); results by rank."""
    hub = fd.LoopbackHub(nranks)
    out, errs = [None] * nranks, []

    def body(r):
        try:
            torch.cuda.set_device(0)
            st = torch.cuda.Stream()
            with torch.cuda.stream(st):
                ctx = fd.Context(0, stream=st.cuda_stream, hub=hub, rank=r)
                try:
                    out[r] = fn(ctx, r)
                    st.synchronize()
                finally:
                    ctx.close()
        except BaseException as e:  # noqa: BLE001
            errs.append((r, e))

    ths = [threading.Thread(target=body, args=(r,), daemon=True) for r in range(nranks)]
    for t in ths:
        t.start()
    for t in ths:
        t.join(timeout)
    assert not any(t.is_alive() for t in ths), "a rank hung"
    hub.close()
    if errs:
        raise errs[0][1]
    return out


def slab_rows(n_last, nranks, r, inner):
    b, e = fd.partition(n_last, nranks, r)
    return b * inner, e * inner


# ----------------------------------------------------------------------------- FD apply

@pytest.mark.parametrize("ns,nranks", [((17, 19, 23), 2), ((17, 19, 23), 3), ((33, 35, 16), 8), ((5, 6, 3), 4),
                                       ((40, 37), 3), ((64, 64, 64), 4), ((131, 131, 131), 8), ((9, 7), 8)])
def test_sharded_fd_apply_matches_oracle(ns, nranks):
    rng = np.random.default_rng(sum(ns) + nranks)
    f = fastdiag.factors_from_eig([rng.standard_normal((n, n)) for n in ns], [rng.uniform(1, 100, n) for n in ns])
    r = rng.standard_normal(int(np.prod(ns)))
    inner = int(np.prod(ns[:-1]))

    def work(ctx, rank):
        plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
        lo, hi = slab_rows(ns[-1], nranks, rank, inner)
        assert plan.N == hi - lo
        x = torch.from_numpy(r[lo:hi].copy()).to(DEV)
        s = torch.empty_like(x)
        fd.fd_apply(plan, x, s)
        fd.fd_apply(plan, x, x)  # aliasing
        torch.cuda.current_stream().synchronize()
        res = (s.cpu().numpy(), x.cpu().numpy())
        plan.close()
        return res

    parts = run_ranks(nranks, work)
    expect = fastdiag.apply(f, r)
    assert rel(np.concatenate([p[0] for p in parts]), expect) <= 1e-12
    np.testing.assert_array_equal(np.concatenate([p[1] for p in parts]), np.concatenate([p[0] for p in parts]))


@pytest.mark.parametrize("ns,nranks", [((17, 19, 23), 2), ((33, 35, 16), 8), ((5, 6, 3), 4), ((40, 24, 64), 3)])
def test_sharded_int8_fd_apply_matches_oracle(ns, nranks, monkeypatch):
    # the int8-split tensor-core mode products on the slab layout and on the transposed
    # mode-3 chunk (with the Lambda divide offset by the chunk start q0), forced onto small shapes
    monkeypatch.setenv("FDIGA_FD_OZ", "1")
    rng = np.random.default_rng(sum(ns) + 10 * nranks)
    f = fastdiag.factors_from_eig([rng.standard_normal((n, n)) for n in ns], [rng.uniform(1, 100, n) for n in ns])
    r = rng.standard_normal(int(np.prod(ns)))
    inner = int(np.prod(ns[:-1]))

    def work(ctx, rank):
        plan = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
        assert plan.path()[0] == "int8_split"
        lo, hi = slab_rows(ns[-1], nranks, rank, inner)
        x = torch.from_numpy(r[lo:hi].copy()).to(DEV)
        s = torch.empty_like(x)
        fd.fd_apply(plan, x, s)
        torch.cuda.current_stream().synchronize()
        res = s.cpu().numpy()
        plan.close()
        return res

    parts = run_ranks(nranks, work)
    assert rel(np.concatenate(parts), fastdiag.apply(f, r)) <= 1e-12


def test_sharded_fd_setup_broadcasts_rank0_factors():
    # every rank runs the cuSOLVER setup; the plan then holds rank 0's factors bit for bit
    _, M, K, _ = splines.colloc_1d(40, 3)

    def work(ctx, rank):
        plan = fd.fd_setup(ctx, [M] * 3, [K] * 3)
        f = [plan.factors(l) for l in range(3)]
        plan.close()
        return f

    fs = run_ranks(3, work)
    for l in range(3):
        for k in range(4):
            np.testing.assert_array_equal(fs[0][l][k], fs[1][l][k])
            np.testing.assert_array_equal(fs[0][l][k], fs[2][l][k])


# ----------------------------------------------------------------------------- matvec with halos

@pytest.mark.parametrize("cfg,ne,nranks", [(3, 6, 2), (3, 9, 3), (5, 7, 5), (5, 4, 3), (3, 3, 4), (5, 16, 8)])
def test_sharded_matvec_matches_oracle(cfg, ne, nranks):
    # cfg5 at ne=7: n=10 planes over 5 ranks, halo p-1 = 4 planes -> halos span several ranks
    c = get_config(cfg)
    disc = assembly.Discretisation(c.d, c.p, ne, c.geometry, c.geo_params)
    x = np.random.default_rng(ne * 10 + nranks).standard_normal(disc.N)
    n = disc.n
    inner = n * n

    def work(ctx, rank):
        A = fd.colloc_assemble(ctx, 3, c.p, ne, c.geometry, c.geo_params)
        lo, hi = slab_rows(n, nranks, rank, inner)
        assert A.N == hi - lo
        y = torch.empty(hi - lo, dtype=torch.float64, device=DEV)
        fd.stencil_matvec(A, torch.from_numpy(x[lo:hi].copy()).to(DEV), y)
        torch.cuda.current_stream().synchronize()
        out = y.cpu().numpy()
        A.close()
        return out

    y = np.concatenate(run_ranks(nranks, work))
    assert rel(y, disc.matvec(x)) <= 1e-12


# ----------------------------------------------------------------------------- GMRES

@pytest.mark.parametrize("cfg,nranks,orth", [(3, 2, 2), (3, 4, 1), (3, 4, 2), (5, 8, 2), (5, 8, 0)])
def test_sharded_gmres_iterations_match_oracle(cfg, nranks, orth):
    c = get_config(cfg)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    n = M.shape[0]
    b = rhs(cfg, n ** 3)

    def work(ctx, rank):
        A = fd.colloc_assemble(ctx, 3, c.p, c.ne, c.geometry, c.geo_params)
        P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
        lo, hi = slab_rows(n, nranks, rank, n * n)
        bt = torch.from_numpy(b[lo:hi].copy()).to(DEV)
        x = torch.empty_like(bt)
        rep = fd.gmres_solve(ctx, A, P, bt, x, orth=orth)
        torch.cuda.current_stream().synchronize()
        if orth == fd.ORTH_DCGS2:  # the profiled solve: same decisions, the collectives charged to t_comm
            xp = torch.empty_like(bt)
            rp = fd.gmres_solve(ctx, A, P, bt, xp, orth=orth, profile=True)
            assert rp["iters"] == rep["iters"] and rp["t_comm_ms"] > 0 and rp["t_fd_ms"] > 0
            parts = sum(rp[k] for k in ("t_fd_ms", "t_matvec_ms", "t_orth_ms", "t_comm_ms", "t_other_ms"))
            assert abs(parts - rp["t_total_ms"]) <= 0.02 * rp["t_total_ms"] + 0.01
        out = (rep, x.cpu().numpy())
        P.close()
        A.close()
        return out

    res = run_ranks(nranks, work)
    reps = [r[0] for r in res]
    ref = GOLD["configs"][str(cfg)]
    assert all(r["iters"] == reps[0]["iters"] for r in reps)          # every rank took the same decisions
    assert all(r["rel_res_true"] == reps[0]["rel_res_true"] for r in reps)
    assert reps[0]["converged"] and abs(reps[0]["iters"] - ref["iters"]) <= 1, (reps[0], ref)
    assert reps[0]["rel_res_true"] <= 1e-8
    x = np.concatenate([r[1] for r in res])
    disc = assembly.Discretisation(3, c.p, c.ne, c.geometry, c.geo_params)
    assert np.linalg.norm(b - disc.matvec(x)) / np.linalg.norm(b) <= 2e-8


# ----------------------------------------------------------------------------- NCCL transport, one rank

@pytest.fixture(scope="module")
def nccl_ctx():
    """A one-rank NCCL communicator: the sharded code path with NCCL self send/recv and all-reduce
    (GMRES captures them in its CUDA graph), i.e. every NCCL call the multi-GPU run issues."""
    uid = fd.nccl_unique_id()
    c = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream, nranks=1, rank=0, nccl_unique_id=uid)
    yield c
    c.close()


def test_nccl_one_rank_fd_apply_and_matvec(nccl_ctx):
    ns = (33, 35, 37)
    rng = np.random.default_rng(7)
    f = fastdiag.factors_from_eig([rng.standard_normal((n, n)) for n in ns], [rng.uniform(1, 100, n) for n in ns])
    plan = fd.fd_setup_from_factors(nccl_ctx, f.U, f.W, f.lam)
    r = rng.standard_normal(int(np.prod(ns)))
    s = torch.empty(r.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, torch.from_numpy(r).to(DEV), s)
    torch.cuda.synchronize()
    assert rel(s.cpu().numpy(), fastdiag.apply(f, r)) <= 1e-12
    c = get_config(5)
    disc = assembly.Discretisation(3, c.p, 6, c.geometry, c.geo_params)
    A = fd.colloc_assemble(nccl_ctx, 3, c.p, 6, c.geometry, c.geo_params)
    x = rng.standard_normal(disc.N)
    y = torch.empty(disc.N, dtype=torch.float64, device=DEV)
    fd.stencil_matvec(A, torch.from_numpy(x).to(DEV), y)
    torch.cuda.synchronize()
    assert rel(y.cpu().numpy(), disc.matvec(x)) <= 1e-12
    plan.close()
    A.close()


def test_nccl_one_rank_int8_fd_apply(nccl_ctx, monkeypatch):
    monkeypatch.setenv("FDIGA_FD_OZ", "1")
    ns = (33, 35, 37)
    rng = np.random.default_rng(8)
    f = fastdiag.factors_from_eig([rng.standard_normal((n, n)) for n in ns], [rng.uniform(1, 100, n) for n in ns])
    plan = fd.fd_setup_from_factors(nccl_ctx, f.U, f.W, f.lam)
    assert plan.path()[0] == "int8_split"
    r = rng.standard_normal(int(np.prod(ns)))
    s = torch.empty(r.size, dtype=torch.float64, device=DEV)
    fd.fd_apply(plan, torch.from_numpy(r).to(DEV), s)
    torch.cuda.synchronize()
    assert rel(s.cpu().numpy(), fastdiag.apply(f, r)) <= 1e-12
    plan.close()


@pytest.mark.parametrize("orth", [1, 2])
def test_nccl_one_rank_gmres_captured(nccl_ctx, orth):
    c = get_config(3)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    A = fd.colloc_assemble(nccl_ctx, 3, c.p, c.ne, c.geometry, c.geo_params)
    P = fd.fd_setup(nccl_ctx, [M] * 3, [K] * 3)
    b = torch.from_numpy(rhs(3, A.N)).to(DEV)
    x = torch.empty_like(b)
    for _ in range(2):  # second solve replays the cached graph
        rep = fd.gmres_solve(nccl_ctx, A, P, b, x, orth=orth)
        assert rep["converged"] and abs(rep["iters"] - GOLD["configs"]["3"]["iters"]) <= 1
        assert rep["rel_res_true"] <= 1e-8
    P.close()
    A.close()


@pytest.mark.parametrize("cfg,nranks", [(3, 3), (5, 4)])
def test_sharded_bicgstab_matches_oracle_counts(cfg, nranks):
    c = get_config(cfg)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    n = M.shape[0]
    b = rhs(cfg, n ** 3)

    def work(ctx, rank):
        A = fd.colloc_assemble(ctx, 3, c.p, c.ne, c.geometry, c.geo_params)
        P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
        lo, hi = slab_rows(n, nranks, rank, n * n)
        bt = torch.from_numpy(b[lo:hi].copy()).to(DEV)
        x = torch.empty_like(bt)
        rep = fd.bicgstab_solve(ctx, A, P, bt, x)
        torch.cuda.current_stream().synchronize()
        out = (rep, x.cpu().numpy())
        P.close()
        A.close()
        return out

    res = run_ranks(nranks, work)
    reps = [r[0] for r in res]
    assert all(r["iters"] == reps[0]["iters"] and r["rel_res_true"] == reps[0]["rel_res_true"] for r in reps)
    assert reps[0]["converged"]
    assert abs(reps[0]["iters"] - GOLD["configs"][str(cfg)]["bicgstab_iters"]) <= 1.0
    x = np.concatenate([r[1] for r in res])
    disc = assembly.Discretisation(3, c.p, c.ne, c.geometry, c.geo_params)
    assert np.linalg.norm(b - disc.matvec(x)) / np.linalg.norm(b) <= 2e-8


def test_nccl_one_rank_bicgstab_captured(nccl_ctx):
    c = get_config(3)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    A = fd.colloc_assemble(nccl_ctx, 3, c.p, c.ne, c.geometry, c.geo_params)
    P = fd.fd_setup(nccl_ctx, [M] * 3, [K] * 3)
    b = torch.from_numpy(rhs(3, A.N)).to(DEV)
    x = torch.empty_like(b)
    rep = fd.bicgstab_solve(nccl_ctx, A, P, b, x)
    assert rep["converged"] and abs(rep["iters"] - GOLD["configs"]["3"]["bicgstab_iters"]) <= 1.0
    P.close()
    A.close()


@pytest.mark.parametrize("cfg,ne,nranks", [(5, 7, 5), (3, 20, 3), (5, 16, 4)])
def test_sharded_matrix_free_matvec(cfg, ne, nranks):
    c = get_config(cfg)
    disc = assembly.Discretisation(c.d, c.p, ne, c.geometry, c.geo_params)
    x = np.random.default_rng(ne + 7 * nranks).standard_normal(disc.N)
    n = disc.n

    def work(ctx, rank):
        A = fd.colloc_assemble(ctx, 3, c.p, ne, c.geometry, c.geo_params, matrix_free=True)
        lo, hi = slab_rows(n, nranks, rank, n * n)
        y = torch.empty(hi - lo, dtype=torch.float64, device=DEV)
        fd.stencil_matvec(A, torch.from_numpy(x[lo:hi].copy()).to(DEV), y)
        torch.cuda.current_stream().synchronize()
        out = y.cpu().numpy()
        A.close()
        return out

    y = np.concatenate(run_ranks(nranks, work))
    assert rel(y, disc.matvec(x)) <= 1e-12


def test_sharded_wq_matvec():
    from oracle import quadrature
    disc = quadrature.WQDiscretisation(3, 3, 7, 3, (1.0, 2.0, 1.0))
    Ao = disc.assemble_wq()
    x = np.random.default_rng(3).standard_normal(disc.N)
    n = disc.n

    def work(ctx, rank):
        A = fd.wq_assemble(ctx, 3, 3, 7, 3, (1.0, 2.0, 1.0))
        lo, hi = slab_rows(n, 3, rank, n * n)
        y = torch.empty(hi - lo, dtype=torch.float64, device=DEV)
        fd.stencil_matvec(A, torch.from_numpy(x[lo:hi].copy()).to(DEV), y)
        torch.cuda.current_stream().synchronize()
        out = y.cpu().numpy()
        A.close()
        return out

    y = np.concatenate(run_ranks(3, work))
    assert rel(y, Ao @ x) <= 1e-12


def test_sharded_gmres_more_ranks_than_planes():
    # cfg3 geometry with ne = 2 (n = 3 planes) over 5 ranks: two ranks own no rows but take part in
    # every collective
    _, M, K, _ = splines.colloc_1d(2, 3)
    n = M.shape[0]
    b = rhs(3, n ** 3, rep=2)

    def work(ctx, rank):
        A = fd.colloc_assemble(ctx, 3, 3, 2, 2, (0.1,))
        P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
        lo, hi = slab_rows(n, 5, rank, n * n)
        bt = torch.from_numpy(b[lo:hi].copy()).to(DEV)
        x = torch.empty_like(bt)
        rep = fd.gmres_solve(ctx, A, P, bt, x, rtol=1e-10)
        torch.cuda.current_stream().synchronize()
        out = (rep, x.cpu().numpy())
        P.close()
        A.close()
        return out

    res = run_ranks(5, work)
    assert all(r[0]["converged"] and r[0]["iters"] == res[0][0]["iters"] for r in res)
    disc = assembly.Discretisation(3, 3, 2, 2, (0.1,))
    x = np.concatenate([r[1] for r in res])
    assert np.linalg.norm(b - disc.matvec(x)) / np.linalg.norm(b) <= 1e-9

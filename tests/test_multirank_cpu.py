"""Multi-process (gloo, CPU) tests of the slab-sharded path's host-side logic.

The library's exchange schedules -- fdiga_transpose_plan (the FD mode-d slab <-> chunk transpose) and
fdiga_halo_plan (the matvec halo planes) -- are host-only C functions; here world_size 2 and 3 real
processes compute them for their own rank, check that every send meets a receive of the same size on
the peer, and then move real data with torch.distributed (gloo) point-to-point messages exactly as
the schedule says.  The local arithmetic between the exchanges is plain numpy, and the assembled
result must equal the oracle's unsharded FD apply / matvec.  No GPU is involved.
"""
import os
import socket
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _exchange(sends, recvs):
    """Point-to-point messages (peer, tensor); self messages are local copies."""
    me = dist.get_rank()
    reqs = []
    local = {}
    for peer, t in sends:
        if peer == me:
            local[peer] = t
        elif t.numel():
            reqs.append(dist.isend(t, peer))
    for peer, t in recvs:
        if peer == me:
            t.copy_(local[peer])
        elif t.numel():
            reqs.append(dist.irecv(t, peer))
    for r in reqs:
        r.wait()


def _fd_case(rank, world, ns):
    import paper_1705_04384_b200 as fd
    from oracle import fastdiag
    d = len(ns)
    rng = np.random.default_rng(11)
    f = fastdiag.factors_from_eig([rng.standard_normal((n, n)) for n in ns], [rng.uniform(1, 100, n) for n in ns])
    r = rng.standard_normal(int(np.prod(ns)))
    nd, Nin = ns[-1], int(np.prod(ns[:-1]))
    o, e = fd.partition(nd, world, rank)
    q0, q1 = fd.partition(Nin, world, rank)
    c, ln = e - o, q1 - q0
    so, sc, to, tc = fd.transpose_plan(Nin, nd, world, rank)
    # the schedule is consistent: what I send to q is what q expects from me
    plans = [None] * world
    dist.all_gather_object(plans, (sc.tolist(), tc.tolist()))
    for q in range(world):
        assert plans[rank][0][q] == plans[q][1][rank], "forward transpose sizes disagree"
    assert sum(sc) == c * Nin and sum(tc) == nd * ln
    # local forward modes 1..d-1 on the slab
    X = r[o * Nin:e * Nin].reshape([c] + [ns[l] for l in range(d - 2, -1, -1)])
    for l in range(d - 1):
        ax = X.ndim - 1 - l
        X = np.moveaxis(np.tensordot(f.W[l], X, axes=([1], [ax])), 0, ax)
    X = X.reshape(c, Nin)
    stage = np.zeros(max(1, c * Nin))
    for q in range(world):
        qb, qe = fd.partition(Nin, world, q)
        stage[so[q]:so[q] + sc[q]] = X[:, qb:qe].reshape(-1)
    st_t = torch.from_numpy(stage)
    T_t = torch.zeros(max(1, nd * ln), dtype=torch.float64)
    _exchange([(q, st_t[so[q]:so[q] + sc[q]]) for q in range(world)],
              [(q, T_t[to[q]:to[q] + tc[q]]) for q in range(world)])
    # mode-d sandwich on T(n_d x len) with the eigenvalue divide
    T = T_t.numpy()[:nd * ln].reshape(nd, ln)
    lam_in = fastdiag.lambda_sum(fastdiag.FDFactors(f.U[:-1], f.W[:-1], f.lam[:-1]))[q0:q1] if d > 1 else 0
    T = f.U[-1] @ ((f.W[-1] @ T) / (f.lam[-1][:, None] + lam_in[None, :]))
    T_t[:nd * ln] = torch.from_numpy(T.reshape(-1))
    _exchange([(q, T_t[to[q]:to[q] + tc[q]]) for q in range(world)],
              [(q, st_t[so[q]:so[q] + sc[q]]) for q in range(world)])
    Y = np.zeros((c, Nin))
    for q in range(world):
        qb, qe = fd.partition(Nin, world, q)
        Y[:, qb:qe] = st_t.numpy()[so[q]:so[q] + sc[q]].reshape(c, qe - qb)
    Y = Y.reshape([c] + [ns[l] for l in range(d - 2, -1, -1)])
    for l in range(d - 2, -1, -1):
        ax = Y.ndim - 1 - l
        Y = np.moveaxis(np.tensordot(f.U[l], Y, axes=([1], [ax])), 0, ax)
    parts = [None] * world
    dist.all_gather_object(parts, Y.reshape(-1))
    if rank == 0:
        s = np.concatenate(parts)
        ref = fastdiag.apply(f, r)
        err = np.linalg.norm(s - ref) / np.linalg.norm(ref)
        assert err <= 1e-12, err


def _halo_case(rank, world, cfg, ne):
    import paper_1705_04384_b200 as fd
    from oracle import assembly
    from synth import get_config
    c = get_config(cfg)
    disc = assembly.Discretisation(3, c.p, ne, c.geometry, c.geo_params)
    n = disc.n
    plane = n * n
    st, wd = fd.colloc_1d_windows(c.p, ne)
    lo, hi, sb, se, rb, re = fd.halo_plan(st, wd, world, rank)
    plans = [None] * world
    dist.all_gather_object(plans, (sb.tolist(), se.tolist(), rb.tolist(), re.tolist()))
    for q in range(world):
        assert (plans[rank][0][q], plans[rank][1][q]) == (plans[q][2][rank], plans[q][3][rank]) or \
            (plans[rank][1][q] <= plans[rank][0][q] and plans[q][3][rank] <= plans[q][2][rank])
    o, e = fd.partition(n, world, rank)
    x = np.random.default_rng(5).standard_normal(disc.N)
    xl = torch.from_numpy(x[o * plane:e * plane].copy())
    ext = torch.zeros((hi - lo) * plane, dtype=torch.float64)
    ext[(o - lo) * plane:(e - lo) * plane] = xl
    sends = [(q, xl[(sb[q] - o) * plane:(se[q] - o) * plane].contiguous()) for q in range(world)
             if q != rank and se[q] > sb[q]]
    recvs = [(q, ext[(rb[q] - lo) * plane:(re[q] - lo) * plane]) for q in range(world)
             if q != rank and re[q] > rb[q]]
    _exchange(sends, recvs)
    A = disc.assemble_csr().tocsr()[o * plane:e * plane]
    # the rows of the slab read only the planes [lo, hi) ...
    cols = A.indices
    if cols.size:
        assert cols.min() >= lo * plane and cols.max() < hi * plane
    # ... and the halo carries exactly the neighbours' values
    np.testing.assert_array_equal(ext.numpy(), x[lo * plane:hi * plane])
    y = A[:, lo * plane:hi * plane] @ ext.numpy()
    parts = [None] * world
    dist.all_gather_object(parts, y)
    if rank == 0:
        yy = np.concatenate(parts)
        ref = disc.matvec(x)
        assert np.linalg.norm(yy - ref) / np.linalg.norm(ref) <= 1e-12


def _worker(rank, world, port, case, args):
    sys.path.insert(0, ROOT)
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        {"fd": _fd_case, "halo": _halo_case}[case](rank, world, *args)
        dist.barrier()
    finally:
        dist.destroy_process_group()


def _run(world, case, *args):
    mp.spawn(_worker, args=(world, _free_port(), case, args), nprocs=world, join=True)


@pytest.mark.parametrize("world,ns", [(2, (6, 7, 9)), (3, (5, 8, 4)), (2, (12, 5)), (3, (4, 4, 2))])
def test_sharded_fd_schedule_gloo(world, ns):
    _run(world, "fd", ns)


@pytest.mark.parametrize("world,cfg,ne", [(2, 3, 5), (3, 5, 7), (2, 5, 4)])
def test_sharded_halo_schedule_gloo(world, cfg, ne):
    _run(world, "halo", cfg, ne)

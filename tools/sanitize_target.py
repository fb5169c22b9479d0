"""Small workload for compute-sanitizer (racecheck / synccheck / memcheck): the hand-rolled mbarrier / TMA /
tcgen05 pipelines at sizes that finish under the sanitizer -- one int8-split FD apply (oz_split + oz_gemm, CTA
pairs, K = 200 and K = 320 (two launches)), one DMMA apply, a GMRES(30) solve with the TMA-streamed DCGS2
Arnoldi passes and a matrix-free BiCGStab solve.  Checks the results against the oracle so that a race that
corrupts data also fails here."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from oracle import fastdiag, splines  # noqa: E402
from synth import get_config, rhs  # noqa: E402

ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(0)
for ns in ((200, 24, 200), (320, 8, 16)):
    U = [rng.standard_normal((n, n)) for n in ns]
    f = fastdiag.factors_from_eig(U, [rng.uniform(1, 100, n) for n in ns])
    P = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    x = rng.standard_normal(int(np.prod(ns)))
    ref = fastdiag.apply(f, x)
    for path in ("int8_split", "dmma"):
        P.set_path(path)
        s = torch.empty(x.size, dtype=torch.float64, device="cuda")
        fd.fd_apply(P, torch.from_numpy(x).cuda(), s)
        torch.cuda.synchronize()
        err = np.linalg.norm(s.cpu().numpy() - ref) / np.linalg.norm(ref)
        print(f"fd_apply {ns} {path}: rel err {err:.2e}", flush=True)
        assert err < 1e-12
    P.close()
c = get_config(3)
ne = 10
_, M, K, _ = splines.colloc_1d(ne, c.p)
for mf in (False, True):
    A = fd.colloc_assemble(ctx, 3, c.p, ne, c.geometry, c.geo_params, matrix_free=mf)
    P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
    b = torch.from_numpy(rhs(3, A.N)).cuda()
    x = torch.empty_like(b)
    r = fd.gmres_solve(ctx, A, P, b, x)
    rb = fd.bicgstab_solve(ctx, A, P, b, x)
    print(f"matrix_free={mf}: gmres {r['iters']} it rel {r['rel_res_true']:.1e}; bicgstab {rb['iters']} it", flush=True)
    assert r["converged"] and rb["converged"]
    P.close()
    A.close()
print("sanitize target ok")

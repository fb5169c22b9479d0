"""Small driver for ncu: FD applies (cfg4 n=256 and cfg5 n=131), cfg5 matvecs and one cfg5 GMRES solve."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector, get_config, rhs  # noqa: E402

what = sys.argv[1] if len(sys.argv) > 1 else "all"
dev = torch.device("cuda:0")
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
if what in ("all", "fd"):
    rng, U, lam = fd_sweep_factors(256)
    plan = fd.fd_setup_from_eig(ctx, U, lam)
    x = torch.from_numpy(fd_sweep_vector(rng, 256 ** 3)).to(dev)
    s = torch.empty_like(x)
    for _ in range(3):
        fd.fd_apply(plan, x, s)
    torch.cuda.synchronize()
    plan.close()
if what in ("all", "cfg5"):
    c = get_config(5)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
    M, K = fd.colloc_1d_factors(c.p, c.ne)
    P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
    b = torch.from_numpy(rhs(5, A.N)).to(dev)
    x = torch.empty_like(b)
    for _ in range(2):
        fd.stencil_matvec(A, b, x)
        fd.fd_apply(P, b, x)
    rep = fd.gmres_solve(ctx, A, P, b, x)
    torch.cuda.synchronize()
    print("cfg5 iters", rep["iters"], "ms", rep["t_total_ms"])
print("launches", ctx.kernel_launches())

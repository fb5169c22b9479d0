"""Time-to-tolerance of FD-preconditioned GMRES(30) on a config (default cfg5, matrix-free operator)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import get_config, rhs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
mf = (sys.argv[2] != "stored") if len(sys.argv) > 2 else True
c = get_config(cfg)
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=mf and c.d == 3)
M, K = fd.colloc_1d_factors(c.p, c.ne)
P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
b = torch.from_numpy(rhs(cfg, A.N)).cuda()
x = torch.empty_like(b)
ts = []
for r in range(6):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    rep = fd.gmres_solve(ctx, A, P, b, x)
    e1.record()
    e1.synchronize()
    if r >= 2:
        ts.append(e0.elapsed_time(e1))
print(f"cfg{cfg} mf={mf}: {sorted(ts)[len(ts) // 2]:.3f} ms (median of {len(ts)}), iters {rep['iters']}")

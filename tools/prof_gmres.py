"""ncu driver: one preconditioned GMRES solve of a BASELINE config (after one warm-up solve)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import get_config, rhs  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
dev = torch.device("cuda:0")
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
c = get_config(cfg)
A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
M, K = fd.colloc_1d_factors(c.p, c.ne)
P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
b = torch.from_numpy(rhs(cfg, A.N)).to(dev)
x = torch.empty_like(b)
for _ in range(2):
    rep = fd.gmres_solve(ctx, A, P, b, x)
torch.cuda.synchronize()
print("cfg", cfg, "iters", rep["iters"], "ms", rep["t_total_ms"])

"""One preconditioned solve on a config (for ncu launch lists):
  python tools/solve_once.py --cfg 5 [--solver gmres|bicgstab] [--matrix-free] [--reps 2]"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import get_config, rhs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, default=5)
ap.add_argument("--solver", default="gmres")
ap.add_argument("--matrix-free", action="store_true")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--orth", type=int, default=2)
a = ap.parse_args()
c = get_config(a.cfg)
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=a.matrix_free)
M, K = fd.colloc_1d_factors(c.p, c.ne)
P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
b = torch.from_numpy(rhs(a.cfg, A.N)).cuda()
x = torch.empty_like(b)
solve = fd.gmres_solve if a.solver == "gmres" else fd.bicgstab_solve
for it in range(a.reps):
    if it == a.reps - 1:
        torch.cuda.synchronize()
        torch.cuda.profiler.start()  # ncu --profile-from-start off: the last solve only
    rep = solve(ctx, A, P, b, x, orth=a.orth) if a.solver == "gmres" else solve(ctx, A, P, b, x)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print(a, rep)

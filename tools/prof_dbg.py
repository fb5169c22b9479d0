import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1705_04384_b200 as fd
from synth import get_config, rhs
from oracle import splines
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
cfg = int(sys.argv[1]); mf = sys.argv[2] == "1"; order = sys.argv[3]
c = get_config(cfg)
A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=mf)
_, M, K, _ = splines.colloc_1d(c.ne, c.p)
P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
b = torch.from_numpy(rhs(cfg, A.N)).cuda()
x = torch.empty_like(b)
for o in order:
    try:
        r = fd.gmres_solve(ctx, A, P, b, x, profile=(o == "p"))
        print(o, r["iters"], {k: round(v, 3) for k, v in r.items() if k.startswith("t_")}, flush=True)
    except Exception as e:
        print(o, "ERROR", e, flush=True)
        break
# follow-up probes after the sequence
try:
    torch.cuda.synchronize()
    print("torch sync ok; torch op", float(torch.ones(3, device="cuda").sum()), flush=True)
except Exception as e:
    print("torch error", e, flush=True)
try:
    y = torch.empty_like(b)
    fd.stencil_matvec(A, b, y)
    torch.cuda.synchronize()
    print("matvec ok", flush=True)
    fd.fd_apply(P, b, y)
    torch.cuda.synchronize()
    print("fd_apply ok", flush=True)
except Exception as e:
    print("lib error", e, flush=True)

"""int8-split FD with streamed factor digits (K > 256) against DMMA: n = 384, 512 and mixed shapes."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402

ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)


def timed(f, reps=5):
    for _ in range(2):
        f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


for ns in [(300, 40, 36), (256, 256, 512), (384, 384, 384), (512, 512, 512)]:
    rng = np.random.default_rng(7)
    U = [rng.standard_normal((n, n)) for n in ns]
    lam = [rng.uniform(1, 100, n) for n in ns]
    os.environ["FDIGA_FD_OZ"] = "0"
    P0 = fd.fd_setup_from_eig(ctx, U, lam)
    os.environ["FDIGA_FD_OZ"] = "1"
    P1 = fd.fd_setup_from_eig(ctx, U, lam)
    assert P1.path()[0] == "int8_split"
    N = int(np.prod(ns))
    x = torch.randn(N, dtype=torch.float64, device="cuda")
    y0 = torch.empty_like(x)
    y1 = torch.empty_like(x)
    fd.fd_apply(P0, x, y0)
    fd.fd_apply(P1, x, y1)
    torch.cuda.synchronize()
    err = float(torch.linalg.norm(y1 - y0) / torch.linalg.norm(y0))
    t0 = timed(lambda: fd.fd_apply(P0, x, y0))
    t1 = timed(lambda: fd.fd_apply(P1, x, y1))
    print(f"n={ns}: rel err {err:.3e}; dmma {t0:.3f} ms, int8 {t1:.3f} ms ({N / t1 / 1e6:.2f} GDOF/s)", flush=True)
    if ns == (512, 512, 512):
        print(fd.fd_apply_timed(P1, x, y1))
    P0.close()
    P1.close()

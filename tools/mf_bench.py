"""Time the stored vs matrix-free collocation matvec (CUDA events; optional --cfg / --only-mf)."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import get_config  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cfg", type=int, nargs="*", default=[3, 5])
ap.add_argument("--only-mf", action="store_true")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
for cfg in a.cfg:
    c = get_config(cfg)
    for mf in ((True,) if a.only_mf else (False, True)):
        A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=mf)
        x = torch.randn(A.N, dtype=torch.float64, device="cuda")
        y = torch.empty_like(x)
        for _ in range(3):
            fd.stencil_matvec(A, x, y)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            fd.stencil_matvec(A, x, y)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1) / a.reps
        print(f"cfg{cfg} {'matrix-free' if mf else 'stored'}: {ms:.4f} ms, {A.N / ms / 1e6:.2f} Grows/s, "
              f"{16 * A.N / ms / 1e6 if mf else (8 * A.nnz + 16 * A.N) / ms / 1e6:.0f} GB/s (algorithmic)")
        A.close()

"""Per-configuration FD apply timing and the autotuned tile per mode (FDIGA_VERBOSE=1 prints them)."""
import os
import sys

import numpy as np
import torch

os.environ.setdefault("FDIGA_VERBOSE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402

ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
for n in [int(v) for v in (sys.argv[1:] or ["65", "131", "256", "257"])]:
    rng = np.random.default_rng(n)
    U = [rng.standard_normal((n, n)) for _ in range(3)]
    lam = [rng.uniform(1, 100, n) for _ in range(3)]
    P = fd.fd_setup_from_eig(ctx, U, lam)
    x = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        fd.fd_apply(P, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fd.fd_apply(P, x, y)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"n={n}: {ms:.4f} ms/apply, {P.flops() / ms / 1e9:.2f} TFLOP/s, {n ** 3 / ms / 1e6:.2f} GDOF/s", flush=True)
    P.close()

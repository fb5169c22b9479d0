"""e2e diagnosis: blocking vs streaming host-buffer FD apply at n = 256 over several step counts, plus
per-call wall times of the streaming path (which call stalls)."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(1)
U = [rng.standard_normal((n, n)) for _ in range(3)]
lam = [rng.uniform(1, 100, n) for _ in range(3)]
P = fd.fd_setup_from_eig(ctx, U, lam)
xh = torch.from_numpy(rng.standard_normal(n ** 3)).pin_memory()
sh = torch.empty(n ** 3, dtype=torch.float64).pin_memory()
xn, sn = xh.numpy(), sh.numpy()
for _ in range(3):
    fd.fd_apply_host(P, xn, sn)
t0 = time.perf_counter()
for _ in range(10):
    fd.fd_apply_host(P, xn, sn)
print(f"sync: {(time.perf_counter() - t0) / 10 * 1e3:.3f} ms/step", flush=True)
for steps in (5, 10, 20, 40):
    for _ in range(3):
        fd.fd_apply_host_async(P, xn, sn)
    fd.fd_host_sync(P)
    t0 = time.perf_counter()
    marks = []
    for _ in range(steps):
        fd.fd_apply_host_async(P, xn, sn)
        marks.append(time.perf_counter())
    fd.fd_host_sync(P)
    t1 = time.perf_counter()
    d = np.diff([t0] + marks) * 1e3
    print(f"async {steps}: {(t1 - t0) / steps * 1e3:.3f} ms/step; per-call enqueue ms: "
          f"max {d.max():.3f} median {np.median(d):.3f}", flush=True)

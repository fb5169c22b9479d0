"""A/B timing of the int8-split FD apply at n (default 256) for the libraries named by FDIGA_LIB (one per
process): whole-apply CUDA-event time over 20 applies and the per-kernel split / GEMM durations."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
path = sys.argv[2] if len(sys.argv) > 2 else "int8_split"
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng, U, lam = fd_sweep_factors((n, n, n))
P = fd.fd_setup_from_eig(ctx, U, lam)
P.set_path(path)
x = torch.from_numpy(fd_sweep_vector(rng, n ** 3)).cuda()
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
ks = {}
for _ in range(5):
    for k, t in fd.fd_apply_timed(P, x, y):
        ks.setdefault(k, []).append(t)
seq = [[] for _ in range(64)]
for _ in range(5):
    for i, (k, t) in enumerate(fd.fd_apply_timed(P, x, y)):
        seq[i].append((k, t))
if os.environ.get("OZ_AB_SEQ"):
    print("  per launch (us): " + "  ".join(f"{v[0][0]}:{np.mean([t for _, t in v]) * 1e3:.1f}" for v in seq if v), flush=True)
lib = os.environ.get("FDIGA_LIB", "in-tree")
print(f"{lib} n={n} {path}: {ms:.4f} ms/apply  " +
      "  ".join(f"{k}: {np.mean(v) * 1e3:.1f} us x{len(v) // 5}" for k, v in ks.items()), flush=True)

"""ncu target: FD applies at n = 131 (cfg5 shape) on the DMMA path."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 131
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng = np.random.default_rng(3)
P = fd.fd_setup_from_eig(ctx, [rng.standard_normal((n, n)) for _ in range(3)], [rng.uniform(1, 100, n) for _ in range(3)])
x = torch.randn(n ** 3, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
for _ in range(3):
    fd.fd_apply(P, x, y)
torch.cuda.synchronize()
print(fd.fd_apply_timed(P, x, y))

import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_1705_04384_b200 as fd
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
for n in (64, 256):
    rng = np.random.default_rng(1)
    P = fd.fd_setup_from_eig(ctx, [rng.standard_normal((n, n)) for _ in range(3)], [rng.uniform(1, 100, n) for _ in range(3)])
    x = torch.randn(n**3, dtype=torch.float64, device="cuda"); y = torch.empty_like(x)
    fd.fd_apply(P, x, y); torch.cuda.synchronize()
    try:
        print(n, P.path()[0], fd.fd_apply_timed(P, x, y))
    except Exception as e:
        print(n, "ERR", e)

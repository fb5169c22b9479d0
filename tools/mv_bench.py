"""Time stencil_matvec on configs[2] and configs[4] (cfg3, cfg5); prints GB/s of algorithmic bytes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import get_config  # noqa: E402

ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
for cfg in (3, 5):
    c = get_config(cfg)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params)
    x = torch.randn(A.N, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    for _ in range(3):
        fd.stencil_matvec(A, x, y)
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(20):
        fd.stencil_matvec(A, x, y)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    byts = 8 * A.nnz + 16 * A.N
    print(f"variant={os.environ.get('FDIGA_MV_VARIANT')} cfg{cfg} {ms*1e3:.1f} us {byts/ms/1e6:.0f} GB/s")

"""fd_setup phase times on the bench's GMRES configs (FDIGA_VERBOSE=1 prints LU / geev / W / finish)."""
import os
import sys
import time

os.environ.setdefault("FDIGA_VERBOSE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04384_b200 as fd  # noqa: E402
from synth import get_config  # noqa: E402

ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
for cfg in [int(a) for a in (sys.argv[1:] or ["2", "3", "5", "2"])]:
    c = get_config(cfg)
    M, K = fd.colloc_1d_factors(c.p, c.ne)
    t0 = time.perf_counter()
    P = fd.fd_setup(ctx, [M] * c.d, [K] * c.d)
    print(f"cfg{cfg}: fd_setup {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
    P.close()

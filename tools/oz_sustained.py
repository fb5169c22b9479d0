"""Sustained (power-capped) int8-split FD apply at n: ms per apply over the last `timed` of `warm + timed`
back-to-back applies, with the NVML SM clock and power at the end (A/B via FDIGA_LIB)."""
import os
import sys
import time

import pynvml as nv
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
warm, timed = 800, 400
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng, U, lam = fd_sweep_factors((n, n, n))
P = fd.fd_setup_from_eig(ctx, U, lam)
x = torch.from_numpy(fd_sweep_vector(rng, n ** 3)).cuda()
y = torch.empty_like(x)
nv.nvmlInit()
h = nv.nvmlDeviceGetHandleByIndex(0)
time.sleep(1.0)
for _ in range(warm):
    fd.fd_apply(P, x, y)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(timed):
    fd.fd_apply(P, x, y)
e1.record()
while not e1.query():
    time.sleep(0.05)
    clk, pw = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1000
e1.synchronize()
print(f"{os.environ.get('FDIGA_LIB', 'in-tree')} n={n}: sustained {e0.elapsed_time(e1) / timed:.4f} ms/apply, "
      f"SM {clk} MHz, {pw:.0f} W", flush=True)

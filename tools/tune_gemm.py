"""Generate paper_1705_04384_b200/gemm_table.txt on a B200: autotune the FD mode-product GEMM for every
single-GPU plan shape the tests, smoke() and bench.py create, and write one line per shape
("L M N K inner cfg  # name time").  Run under gpurun; copy gpurun_out/gemm_table.txt into the package."""
import os
import sys

import numpy as np

OUT = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/gemm_table.txt"
os.environ["FDIGA_GEMM_TUNE_ALWAYS"] = "1"
os.environ["FDIGA_GEMM_TABLE_OUT"] = OUT
if os.path.exists(OUT):
    os.remove(OUT)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1705_04384_b200 as fd  # noqa: E402

ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
shapes = [(n, n, n) for n in (65, 128, 131, 256, 257, 512)] + [(257, 257), (32, 32), (256, 256)]
for ns in shapes:
    rng = np.random.default_rng(1)
    U = [np.eye(n) + 0.01 * rng.standard_normal((n, n)) for n in ns]
    lam = [rng.uniform(1, 2, n) for n in ns]
    P = fd.fd_setup_from_eig(ctx, U, lam)
    P.close()
    print(ns, flush=True)
with open(OUT) as fh:
    body = fh.read()
with open(OUT, "w") as fh:
    fh.write("# FD mode-product GEMM tile table (tools/tune_gemm.py on a B200; fd_gemm.cu reads it).\n"
             "# layout M N K inner cfg  # tile, time of the winner\n" + body)
print(body)

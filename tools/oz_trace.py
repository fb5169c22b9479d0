"""In-kernel timeline of CTA pair 0 of the last oz_gemm launch (a FDIGA_OZ_TRACE variant build, tools/variant.sh
<name> - -DFDIGA_OZ_TRACE; run with FDIGA_LIB=scratch/<name>/libfdiga.so).  Cycles relative to the kernel start."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1705_04384_b200 as fd  # noqa: E402
from paper_1705_04384_b200 import _lib  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 256
NPASS = int(os.environ.get("NPASS", "4"))
WPP = 8 // NPASS
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
rng, U, lam = fd_sweep_factors((n, n, n))
P = fd.fd_setup_from_eig(ctx, U, lam)
P.set_path("int8_split")
x = torch.from_numpy(fd_sweep_vector(rng, n ** 3)).cuda()
y = torch.empty_like(x)
for _ in range(3):
    fd.fd_apply(P, x, y)
torch.cuda.synchronize()
lib = ctypes.CDLL(_lib.LIB_PATH)
buf = (ctypes.c_longlong * 4096)()
rc = lib.fdiga_oz_trace_read(buf, 4096)
assert rc == 0, rc
t = np.array(buf[:], dtype=np.int64)
t0 = t[0]
r = lambda v: int(v - t0) if v else -1
print(f"setup done {r(t[1])}  epilogue past last tile {r(t[2])}  fixup done {r(t[3])}  kernel end {r(t[4])}")
ntile = 7
print("MMA warps: per phase q: start | chunk0: wait-begin, planes-ready | chunk1: wait-begin, planes-ready | chunk0 issued | last chunk issued")
for mw in range(2):
    for q in range(ntile * NPASS):
        e = t[16 + mw * 512 + q * 8: 16 + mw * 512 + q * 8 + 8]
        if e[0] == 0:
            continue
        print(f"  mw{mw} q{q:2d} (tile {q // NPASS} pass {q % NPASS}): start {r(e[0]):7d} | {r(e[1]):7d} {r(e[2]):7d} | {r(e[3]):7d} {r(e[4]):7d} | {r(e[5]):7d} | {r(e[6]):7d}")
print("epilogue warp 0: per (q, k): wait-begin, slot complete (waited), drained (drain cycles)")
for q in range(ntile * NPASS):
    for k in range(WPP):
        e = t[2048 + (q * WPP + k) * 4: 2048 + (q * WPP + k) * 4 + 4]
        if e[0] == 0:
            continue
        print(f"  q{q:2d} k{k}: {r(e[0]):7d} {r(e[1]):7d} (+{int(e[1] - e[0]):6d}) {r(e[2]):7d} (+{int(e[2] - e[1]):5d})")
    if q % NPASS == NPASS - 1:
        e = t[3072 + (q // NPASS) * 4: 3072 + (q // NPASS) * 4 + 4]
        print(f"  tile {q // NPASS}: prolog done {r(e[2])}  store begins {r(e[0])}  stores issued {r(e[1])} (+{int(e[1] - e[0])})")

"""Every FD mode-product tile configuration (forced through FDIGA_GEMM_FORCE_*) against the oracle, on ragged
shapes that exercise partial tiles, odd leading dimensions and the fused divide epilogue."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPT = r'''
import sys, numpy as np, torch
sys.path.insert(0, %r)
import paper_1705_04384_b200 as fd
from oracle import fastdiag
ctx = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
worst = 0.0
for ns in [(19, 24, 33), (64, 64, 64), (131, 7, 40), (33, 65), (72, 16, 145)]:
    rng = np.random.default_rng(sum(ns))
    f = fastdiag.factors_from_eig([rng.standard_normal((n, n)) for n in ns], [rng.uniform(1, 100, n) for n in ns])
    P = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    r = rng.standard_normal(int(np.prod(ns)))
    s = torch.empty(r.size, dtype=torch.float64, device="cuda")
    fd.fd_apply(P, torch.from_numpy(r).cuda(), s)
    e = fastdiag.apply(f, r)
    worst = max(worst, float(np.linalg.norm(s.cpu().numpy() - e) / np.linalg.norm(e)))
    P.close()
print(worst)
''' % ROOT


@pytest.mark.parametrize("cfg", list(range(18)))
def test_forced_gemm_config_matches_oracle(cfg):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, FDIGA_GEMM_FORCE_KN=str(cfg), FDIGA_GEMM_FORCE_NK=str(cfg))
    out = subprocess.run([sys.executable, "-c", SCRIPT], env=env, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    assert float(out.stdout.strip().splitlines()[-1]) <= 1e-12

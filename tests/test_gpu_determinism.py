"""Race detection without compute-sanitizer (closed on this pool): the hand-rolled mbarrier /
TMA / tcgen05 pipelines (oz_gemm's CTA pairs, the TMA-fed Arnoldi passes, the DMMA cp.async rings) are run
many times on the same inputs and must give bit-identical results every time -- a missing wait or a slot
reused too early shows up as run-to-run differences long before it shows up as a wrong answer."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1705_04384_b200 as fd  # noqa: E402
from oracle import fastdiag, splines  # noqa: E402
from synth import fd_sweep_factors, fd_sweep_vector, get_config, rhs  # noqa: E402

DEV = torch.device("cuda:0")


@pytest.fixture(scope="module")
def ctx():
    c = fd.Context(0, stream=torch.cuda.current_stream().cuda_stream)
    yield c
    c.close()


@pytest.mark.parametrize("path", ["int8_split", "dmma"])
@pytest.mark.parametrize("ns", [(256, 256, 256), (200, 72, 320)])
def test_fd_apply_bitwise_repeatable(ctx, ns, path):
    rng, U, lam = fd_sweep_factors(ns)
    f = fastdiag.factors_from_eig(U, lam)
    P = fd.fd_setup_from_factors(ctx, f.U, f.W, f.lam)
    P.set_path(path)
    x = torch.from_numpy(fd_sweep_vector(rng, int(np.prod(ns)))).to(DEV)
    s0 = torch.empty_like(x)
    fd.fd_apply(P, x, s0)
    s = torch.empty_like(x)
    for _ in range(25):
        fd.fd_apply(P, x, s)
        assert torch.equal(s, s0)
    P.close()


@pytest.mark.parametrize("matrix_free", [False, True])
def test_gmres_bitwise_repeatable(ctx, matrix_free):
    c = get_config(5)
    A = fd.colloc_assemble(ctx, c.d, c.p, c.ne, c.geometry, c.geo_params, matrix_free=matrix_free)
    _, M, K, _ = splines.colloc_1d(c.ne, c.p)
    P = fd.fd_setup(ctx, [M] * 3, [K] * 3)
    b = torch.from_numpy(rhs(5, A.N)).to(DEV)
    x0 = torch.empty_like(b)
    r0 = fd.gmres_solve(ctx, A, P, b, x0, history=True)
    x = torch.empty_like(b)
    for _ in range(8):
        r = fd.gmres_solve(ctx, A, P, b, x, history=True)
        assert r["iters"] == r0["iters"] and r["rel_res_true"] == r0["rel_res_true"]
        np.testing.assert_array_equal(r["history"], r0["history"])
        assert torch.equal(x, x0)
    P.close()
    A.close()

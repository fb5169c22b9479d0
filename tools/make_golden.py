"""Write tests/golden/oracle_gmres.json: the ORACLE's GMRES(30)+FD and BiCGStab+FD iteration counts on
the full-size BASELINE.json configs (seeded RHS from synth/).  Calls only oracle/ and synth/
(DESIGN.md §Oracle)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import assembly, fastdiag, krylov  # noqa: E402
from synth import get_config, rhs  # noqa: E402


def main():
    out = {"_source": "tools/make_golden.py: oracle/krylov.gmres (MGS, right-preconditioned, m=30, rtol=1e-8, x0=0) "
                      "and oracle/krylov.bicgstab (right-preconditioned, rtol=1e-8, x0=0, half-iteration counts) "
                      "with oracle/fastdiag on oracle/assembly's sum-factorised operator; b = synth.rhs(cfg, N, rep=0)",
           "configs": {}}
    for cfg in (1, 2, 3, 5):
        c = get_config(cfg)
        t0 = time.time()
        disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
        f = fastdiag.setup([disc.M] * c.d, [disc.K] * c.d)
        b = rhs(cfg, disc.N)
        x, rep = krylov.gmres(disc.matvec, b, precond=lambda v: fastdiag.apply(f, v))
        xb, repb = krylov.bicgstab(disc.matvec, b, precond=lambda v: fastdiag.apply(f, v))
        out["configs"][str(cfg)] = dict(d=c.d, p=c.p, ne=c.ne, n=disc.n, N=disc.N, iters=rep["iters"],
                                        rel_res_true=rep["rel_res_true"], bicgstab_iters=repb["iters"],
                                        bicgstab_rel_res_true=repb["rel_res_true"],
                                        seconds=round(time.time() - t0, 2))
        print(cfg, out["configs"][str(cfg)], flush=True)
    # NEXT-4 convection-diffusion workloads: GMRES(30) with the wind-aware FD preconditioner (collocation
    # analogue of eq:convec_prec_2: K_2 + H_2 in the angular direction, complex pairs allowed) and without
    # the wind (eq:convec_prec_1), max 300 steps
    import numpy as np
    from oracle import splines
    out["next4"] = {}
    for cfg in (6, 7):
        c = get_config(cfg)
        t0 = time.time()
        disc = assembly.Discretisation(c.d, c.p, c.ne, c.geometry, c.geo_params, c.wind, c.wind_params)
        H2 = splines.colloc_1d_convection(c.ne, c.p, 2 * c.wind_params[0] / np.pi)
        fw = fastdiag.setup([disc.M] * 3, [disc.K, disc.K + H2, disc.K], allow_complex=True, cond_max=1e30)
        f0 = fastdiag.setup([disc.M] * 3, [disc.K] * 3)
        b = rhs(cfg, disc.N)
        _, rw = krylov.gmres(disc.matvec, b, precond=lambda v: fastdiag.apply(fw, v), max_iters=300)
        _, r0 = krylov.gmres(disc.matvec, b, precond=lambda v: fastdiag.apply(f0, v), max_iters=300)
        out["next4"][str(cfg)] = dict(ne=c.ne, p=c.p, n=disc.n, N=disc.N, omega=c.wind_params[0],
                                      iters_wind_fd=rw["iters"], converged_wind_fd=rw["converged"],
                                      rel_res_true_wind_fd=rw["rel_res_true"], has_complex_pairs=bool(fw.has_pairs),
                                      iters_plain_fd=r0["iters"], converged_plain_fd=r0["converged"],
                                      seconds=round(time.time() - t0, 2))
        print(cfg, out["next4"][str(cfg)], flush=True)
    # NEXT-3 weighted-quadrature Galerkin workloads: GMRES(30) and BiCGStab with the symmetric FD of the
    # exact 1D Galerkin pencils
    from oracle import quadrature
    out["wq"] = {}
    for cfg in (8, 9):
        c = get_config(cfg)
        t0 = time.time()
        disc = quadrature.WQDiscretisation(c.d, c.p, c.ne, c.geometry, c.geo_params)
        A = disc.assemble_wq()
        M, K, _ = splines.galerkin_1d(c.ne, c.p, 0.0)
        f = fastdiag.setup([M] * c.d, [K] * c.d)
        b = rhs(cfg, disc.N)
        _, rg = krylov.gmres(lambda v: A @ v, b, precond=lambda v: fastdiag.apply(f, v))
        _, rb = krylov.bicgstab(lambda v: A @ v, b, precond=lambda v: fastdiag.apply(f, v))
        out["wq"][str(cfg)] = dict(d=c.d, p=c.p, ne=c.ne, n=disc.n, N=disc.N, nnz=int(A.nnz), iters=rg["iters"],
                                   rel_res_true=rg["rel_res_true"], bicgstab_iters=rb["iters"],
                                   seconds=round(time.time() - t0, 2))
        print(cfg, out["wq"][str(cfg)], flush=True)
    with open(os.path.join(ROOT, "tests", "golden", "oracle_gmres.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()

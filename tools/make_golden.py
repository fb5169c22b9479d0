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
    with open(os.path.join(ROOT, "tests", "golden", "oracle_gmres.json"), "w") as fh:
        json.dump(out, fh, indent=1)


if __name__ == "__main__":
    main()

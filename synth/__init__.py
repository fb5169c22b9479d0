"""Seeded synthetic inputs shared by the oracle side (tests, cpu_baseline) and the
CUDA side (tests, bench, smoke).

This module holds NONE of the method's arithmetic: it only names the five
BASELINE.json configurations and draws the random numbers they call for
(right-hand sides, the cfg4 random factors).  Everything derived from these
draws (knots, Greville points, 1D collocation matrices, eigendecompositions,
inverses, assembled operators) is computed independently by `oracle/` and by
`paper_1705_04384_b200/` (the CUDA library).

Recipe:
  * seeds: numpy.random.default_rng(1000*cfg + rep)   (PCG64)
  * cfg1/2/3/5: b ~ U(-1, 1)^N drawn in flattened order, i_1 fastest
  * cfg4: U_1, U_2, U_3 ~ N(0,1)^{n x n} (row-major), then lam_1, lam_2, lam_3 ~ U(1,100)^n,
          then x ~ N(0,1)^N.
No public dataset is involved: the paper's domains are analytic, and its radii and
right-hand side are unstated (SURVEY.md §4 "Gaps").
"""
from .configs import CONFIGS, Config, get_config, n_dofs  # noqa: F401
from .gen import rng_for, rhs, fd_sweep_factors, fd_sweep_vector  # noqa: F401

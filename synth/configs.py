"""The five BASELINE.json configurations as plain data (no arithmetic of the method).

Geometry ids (shared vocabulary with include/fdiga.h `FDIGA_GEOM_*`):
  0 identity map on [0,1]^d
  1 quarter annulus, radii (r0, r1) = geo_params[0:2]            (2D, "quarter of ring")
  2 deformed cube x_k = xi_k + a*prod_l sin(pi xi_l), a = geo_params[0]   (3D, BASELINE.json configs[2])
  3 thick quarter ring: annulus x height, (r0, r1, height) = geo_params[0:3]  (3D, BASELINE.json configs[4])
"""
from dataclasses import dataclass, field
from typing import Tuple

GEOM_IDENTITY = 0
GEOM_ANNULUS = 1
GEOM_DEFORMED_CUBE = 2
GEOM_THICK_RING = 3


@dataclass(frozen=True)
class Config:
    cfg: int
    d: int
    p: int
    ne: int                  # elements per direction (uniform open knots)
    geometry: int
    geo_params: Tuple[float, ...] = field(default_factory=tuple)
    note: str = ""
    wind: int = 0            # NEXT-4 only: 0 none, 1 constant, 2 rigid rotation about x_3 (omega = wind_params[0])
    wind_params: Tuple[float, ...] = field(default_factory=tuple)

    @property
    def n(self) -> int:
        # n = m - 2 with m = ne + p basis functions per direction
        return self.ne + self.p - 2

    @property
    def N(self) -> int:
        return self.n ** self.d


CONFIGS = {
    1: Config(1, 2, 2, 32, GEOM_IDENTITY, (), "2D p=2 32x32 identity; FD exact => GMRES 1 iteration"),
    2: Config(2, 2, 3, 256, GEOM_ANNULUS, (1.0, 2.0), "2D p=3 256x256 quarter annulus r in [1,2]"),
    3: Config(3, 3, 3, 64, GEOM_DEFORMED_CUBE, (0.1,), "3D p=3 64^3 deformed cube"),
    5: Config(5, 3, 5, 128, GEOM_THICK_RING, (1.0, 2.0, 1.0), "3D p=5 128^3 thick quarter ring"),
}

# NEXT-4 workloads (not BASELINE.json configs): convection-diffusion L_w = -Lap + w . grad
# (eq:convection) on the cfg5 geometry with the rotating wind w = omega (-y, x, 0), for which
# J^{-1} w = (0, 2 omega / pi, 0) exactly, so the univariate wind of eq:convec_prec_2 is w~_2 = 2 omega / pi.
#   6: strongly convective (omega = 3000, ne = 32): the preconditioner's pencil (K_2 + H_2, M_2) has complex
#      pairs; without the wind (eq:convec_prec_1) GMRES(30) does not converge in 300 steps.
#   7: mildly convective (omega = 10) at the full cfg5 size: real spectrum.
NEXT4_CONFIGS = {
    6: Config(6, 3, 5, 32, GEOM_THICK_RING, (1.0, 2.0, 1.0), "NEXT-4: cfg5 geometry, rotating wind omega=3000",
              2, (3000.0,)),
    7: Config(7, 3, 5, 128, GEOM_THICK_RING, (1.0, 2.0, 1.0), "NEXT-4: cfg5 geometry, rotating wind omega=10",
              2, (10.0,)),
}

# NEXT-3 workloads: the weighted-quadrature Galerkin system A_wq u = f (eq:WQsystem)
# with the symmetric FD of the exact 1D Galerkin pencils (eq:univariateWQ) as preconditioner.
#   8: the quarter annulus of cfg2 (Table 3's domain), p = 3, 256 x 256 elements
#   9: the thick quarter ring of cfg5, p = 3, 32^3 elements
WQ_CONFIGS = {
    8: Config(8, 2, 3, 256, GEOM_ANNULUS, (1.0, 2.0), "NEXT-3: WQ-Galerkin, quarter annulus p=3 256x256"),
    9: Config(9, 3, 3, 32, GEOM_THICK_RING, (1.0, 2.0, 1.0), "NEXT-3: WQ-Galerkin, thick ring p=3 32^3"),
}

# cfg4 is the isolated FD-apply sweep: d=3, n in {128, 256, 512}, random factors.
FD_SWEEP_N = (128, 256, 512)


def get_config(cfg: int) -> Config:
    for table in (CONFIGS, NEXT4_CONFIGS, WQ_CONFIGS):
        if cfg in table:
            return table[cfg]
    raise KeyError(cfg)


def n_dofs(ne: int, p: int) -> int:
    return ne + p - 2

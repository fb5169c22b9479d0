"""Seeded draws.  Only random numbers: no knots, no matrices of the method, no inverses."""
import numpy as np


def rng_for(cfg: int, rep: int = 0) -> np.random.Generator:
    """numpy PCG64 stream for config `cfg`, repetition `rep`."""
    return np.random.default_rng(1000 * cfg + rep)


def rhs(cfg: int, N: int, rep: int = 0) -> np.ndarray:
    """b ~ U(-1,1)^N in flattened order (i_1 fastest), float64."""
    return rng_for(cfg, rep).uniform(-1.0, 1.0, size=N)


def fd_sweep_factors(n, rep: int = 0, d: int = 3, seed_cfg: int = 4):
    """cfg4 factors: U_l ~ N(0,1)^{n_l x n_l} for l=1..d, then lam_l ~ U(1,100)^{n_l}.

    `n` is an int (cube) or a length-d sequence (non-cubic weak-scaling family).
    Returns (rng, [U_1..U_d], [lam_1..lam_d]); the rng is returned so that the
    vector x can be drawn next from the same stream (fd_sweep_vector).
    """
    ns = [int(n)] * d if np.isscalar(n) else [int(v) for v in n]
    rng = rng_for(seed_cfg, rep)
    U = [rng.standard_normal((nl, nl)) for nl in ns]
    lam = [rng.uniform(1.0, 100.0, size=nl) for nl in ns]
    return rng, U, lam


def fd_sweep_vector(rng: np.random.Generator, N: int) -> np.ndarray:
    """x ~ N(0,1)^N, drawn after the factors."""
    return rng.standard_normal(N)

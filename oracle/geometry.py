"""Analytic geometry maps F: [0,1]^d -> Omega with Jacobian and Hessians (oracle).

P:154  Omega = F([0,1]^d).  The configurations fix analytic maps (BASELINE.json configs),
so F, J = dF/dxi and H_c = d^2 F_c / dxi^2 are written in closed form.  Each function is
vectorised over an array of parametric points xi of shape (P, d) and returns
  F (P, d),  J (P, d, d) with J[:, c, a] = dF_c/dxi_a,  H (P, d, d, d) with H[:, c, a, b] = d^2F_c/dxi_a dxi_b.

Readings: xi_1 radial, xi_2 angular, xi_3 height (SURVEY.md §8(c) reading 8);
the deformed cube adds the same scalar bump to every coordinate (reading 10).
The inverse maps (used only by the finite-difference pins) are given too.
"""
import numpy as np

IDENTITY, ANNULUS, DEFORMED_CUBE, THICK_RING = 0, 1, 2, 3


def identity(xi):
    P, d = xi.shape
    J = np.broadcast_to(np.eye(d), (P, d, d)).copy()
    H = np.zeros((P, d, d, d))
    return xi.copy(), J, H


def annulus(xi, r0=1.0, r1=2.0):
    """(x, y) = (r cos th, r sin th), r = r0 + (r1-r0) xi_1, th = (pi/2) xi_2."""
    a, b = xi[:, 0], xi[:, 1]
    dr = r1 - r0
    w = np.pi / 2
    r = r0 + dr * a
    th = w * b
    c, s = np.cos(th), np.sin(th)
    P = xi.shape[0]
    F = np.stack([r * c, r * s], axis=1)
    J = np.zeros((P, 2, 2))
    J[:, 0, 0] = dr * c
    J[:, 0, 1] = -r * w * s
    J[:, 1, 0] = dr * s
    J[:, 1, 1] = r * w * c
    H = np.zeros((P, 2, 2, 2))
    # x = r c: d2/da2 = 0, d2/dadb = -dr w s, d2/db2 = -r w^2 c
    H[:, 0, 0, 1] = H[:, 0, 1, 0] = -dr * w * s
    H[:, 0, 1, 1] = -r * w * w * c
    # y = r s: d2/dadb = dr w c, d2/db2 = -r w^2 s
    H[:, 1, 0, 1] = H[:, 1, 1, 0] = dr * w * c
    H[:, 1, 1, 1] = -r * w * w * s
    return F, J, H


def annulus_inverse(x, r0=1.0, r1=2.0):
    r = np.hypot(x[:, 0], x[:, 1])
    th = np.arctan2(x[:, 1], x[:, 0])
    return np.stack([(r - r0) / (r1 - r0), th / (np.pi / 2)], axis=1)


def deformed_cube(xi, amp=0.1):
    """x_k = xi_k + amp * sin(pi xi_1) sin(pi xi_2) sin(pi xi_3), k = 1..3."""
    P = xi.shape[0]
    s = np.sin(np.pi * xi)
    c = np.cos(np.pi * xi)
    g = s[:, 0] * s[:, 1] * s[:, 2]
    dg = np.stack([np.pi * c[:, 0] * s[:, 1] * s[:, 2],
                   np.pi * s[:, 0] * c[:, 1] * s[:, 2],
                   np.pi * s[:, 0] * s[:, 1] * c[:, 2]], axis=1)
    hg = np.zeros((P, 3, 3))
    pi2 = np.pi ** 2
    hg[:, 0, 0] = -pi2 * g
    hg[:, 1, 1] = -pi2 * g
    hg[:, 2, 2] = -pi2 * g
    hg[:, 0, 1] = hg[:, 1, 0] = pi2 * c[:, 0] * c[:, 1] * s[:, 2]
    hg[:, 0, 2] = hg[:, 2, 0] = pi2 * c[:, 0] * s[:, 1] * c[:, 2]
    hg[:, 1, 2] = hg[:, 2, 1] = pi2 * s[:, 0] * c[:, 1] * c[:, 2]
    F = xi + amp * g[:, None]
    J = np.broadcast_to(np.eye(3), (P, 3, 3)) + amp * dg[:, None, :]
    H = np.broadcast_to(amp * hg[:, None, :, :], (P, 3, 3, 3)).copy()
    return F, J, H


def deformed_cube_inverse(x, amp=0.1, iters=60):
    """Newton iteration on F(xi) = x (used only by finite-difference pins)."""
    xi = x.copy()
    for _ in range(iters):
        F, J, _ = deformed_cube(xi, amp)
        xi = xi - np.linalg.solve(J, (F - x)[..., None])[..., 0]
    return xi


def thick_ring(xi, r0=1.0, r1=2.0, height=1.0):
    """(r cos th, r sin th, height*xi_3): the quarter annulus extruded along z."""
    F2, J2, H2 = annulus(xi[:, :2], r0, r1)
    P = xi.shape[0]
    F = np.concatenate([F2, height * xi[:, 2:3]], axis=1)
    J = np.zeros((P, 3, 3))
    J[:, :2, :2] = J2
    J[:, 2, 2] = height
    H = np.zeros((P, 3, 3, 3))
    H[:, :2, :2, :2] = H2
    return F, J, H


def thick_ring_inverse(x, r0=1.0, r1=2.0, height=1.0):
    return np.concatenate([annulus_inverse(x[:, :2], r0, r1), x[:, 2:3] / height], axis=1)


WIND_NONE, WIND_CONSTANT, WIND_ROTATING = 0, 1, 2


def wind(kind: int, x: np.ndarray, params=()):
    """Physical wind w(x) of the convection-diffusion operator L_w = -Lap + w . grad (eq:convection).
    WIND_CONSTANT: w = (w_1..w_d) = params; WIND_ROTATING: w = omega (-x_2, x_1, 0..) (rigid rotation about the
    x_3 axis), omega = params[0].  Returns (P, d)."""
    P, d = x.shape
    if kind == WIND_NONE:
        return np.zeros((P, d))
    if kind == WIND_CONSTANT:
        return np.broadcast_to(np.asarray(params[:d], dtype=np.float64), (P, d)).copy()
    if kind == WIND_ROTATING:
        w = np.zeros((P, d))
        w[:, 0] = -params[0] * x[:, 1]
        w[:, 1] = params[0] * x[:, 0]
        return w
    raise ValueError(f"unknown wind {kind}")


def evaluate(geometry: int, xi: np.ndarray, params=()):
    if geometry == IDENTITY:
        return identity(xi)
    if geometry == ANNULUS:
        return annulus(xi, *params)
    if geometry == DEFORMED_CUBE:
        return deformed_cube(xi, *params)
    if geometry == THICK_RING:
        return thick_ring(xi, *params)
    raise ValueError(f"unknown geometry {geometry}")


def inverse(geometry: int, x: np.ndarray, params=()):
    if geometry == IDENTITY:
        return x.copy()
    if geometry == ANNULUS:
        return annulus_inverse(x, *params)
    if geometry == DEFORMED_CUBE:
        return deformed_cube_inverse(x, *params)
    if geometry == THICK_RING:
        return thick_ring_inverse(x, *params)
    raise ValueError(f"unknown geometry {geometry}")

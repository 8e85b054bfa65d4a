"""Closed-form Stokes layer potentials on the unit sphere (test-only expected values).

Sources (classical Stokes flow, viscosity 1, S and T normalised as in
PAPER.md eqs. (1)-(4), lines 15-31):

* SL of a constant density F (rigid translation; the traction of a
  translating sphere is uniform): (1/8pi) int S F dS =
    (2/3) F                                              |y| <= 1
    (1/2)(F/R + (F.y) y/R^3) + (1/6)(F/R^3 - 3 (F.y) y/R^5)   R = |y| > 1
  (the sphere's translation velocity U = (2/3) F, Stokes' solution).
* SL of f = Omega x x (rigid rotation): (1/3) Omega x y inside/on,
  (1/3) Omega x y / R^3 outside.
* DL of a rigid motion q = U + Omega x x: chi(y) q(y) with chi = 1, 1/2, 0
  inside / on / outside (the DL reproduces rigid motions; PAPER.md:58 fixes chi).
* Green's identity for a Stokes flow u with stress sigma (mu = 1):
  SL[sigma.n] + DL[u] = chi u.  With u = (y2, 0, 0), p = 0:
  sigma.n = (n2, n1, 0) = (x2, x1, 0) on the unit sphere.
"""
from __future__ import annotations

import numpy as np


def sl_translation(F, y):
    F = np.asarray(F, dtype=np.float64)
    R = np.linalg.norm(y, axis=0)
    Fy = F @ y
    inside = np.repeat((2.0 / 3.0 * F)[:, None], y.shape[1], axis=1)
    with np.errstate(divide="ignore", invalid="ignore"):
        outside = 0.5 * (F[:, None] / R + Fy * y / R ** 3) + (1.0 / 6.0) * (F[:, None] / R ** 3 - 3 * Fy * y / R ** 5)
    return np.where(R <= 1.0, inside, outside)


def sl_rotation(Omega, y):
    R = np.linalg.norm(y, axis=0)
    rot = np.cross(np.asarray(Omega, dtype=np.float64), y.T).T / 3.0
    return np.where(R <= 1.0, rot, rot / R ** 3)


def chi_of_b(b):
    return np.where(b < 0, 1.0, np.where(b > 0, 0.0, 0.5))


SHEAR_TRACTION = np.array([[0.0, 1.0, 0.0], [1.0, 0.0, 0.0], [0.0, 0.0, 0.0]])  # (x2, x1, 0)
SHEAR_VELOCITY = np.array([[0.0, 1.0, 0.0], [0.0, 0.0, 0.0], [0.0, 0.0, 0.0]])  # (x2, 0, 0)


def spheroid_translation_velocity(y, n_gauss: int = 400):
    """Velocity of the prolate spheroid x1^2 + 4 x2^2 + 4 x3^2 = 1 translating with (1, 0, 0)
    in fluid at rest (mu = 1), at points y (3, K) outside it: Chwang & Wu's singularity
    solution (J. Fluid Mech. 1975), a line of Stokeslets of constant strength and of potential
    doublets of strength proportional to (c^2 - s^2) on the focal segment |s| <= c = a e,
        u(y) = (A/2) int S(y - s e1) e1 ds - (B/2) int (c^2 - s^2) D(y - s e1) e1 ds,
        S(r) e1 = e1/|r| + r r_1/|r|^3,   D(r) e1 = -e1/|r|^3 + 3 r r_1/|r|^5,
        A = 2 e^2 / (-2e + (1 + e^2) ln((1+e)/(1-e))),  B = (1 - e^2) A / (2 e^2),
    integrated by n_gauss-point Gauss-Legendre (the segment lies inside the body, so the
    integrand is smooth for every exterior y).  Pinned by u = e1 on the surface and by the
    plain quadrature of the single layer at points away from it (tests/test_spheroid.py)."""
    import math

    a, b = 1.0, 0.5
    e = math.sqrt(1.0 - (b / a) ** 2)
    c = a * e
    L = math.log((1.0 + e) / (1.0 - e))
    A = 2.0 * e * e / (-2.0 * e + (1.0 + e * e) * L)
    B = (1.0 - e * e) * A / (2.0 * e * e)
    s, wq = np.polynomial.legendre.leggauss(n_gauss)
    s, wq = c * s, c * wq
    y = np.asarray(y, dtype=np.float64)
    u = np.zeros_like(y)
    for sk, wk in zip(s, wq):
        r = y.copy()
        r[0] -= sk
        R = np.linalg.norm(r, axis=0)
        St = r * (r[0] / R ** 3)
        St[0] += 1.0 / R
        Dt = 3.0 * r * (r[0] / R ** 5)
        Dt[0] -= 1.0 / R ** 3
        u += wk * (0.5 * A * St - 0.5 * B * (c * c - sk * sk) * Dt)
    return u

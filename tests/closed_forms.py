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

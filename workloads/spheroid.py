"""Seeded inputs of the paper's accuracy/timing benchmark (Sec. 4.1):
the Stokeslet integral near the prolate spheroid x1^2 + 4 x2^2 + 4 x3^2 = 1 translating with
velocity (1, 0, 0).

  * surface: Ellipsoid((1, 1/2, 1/2)), the paper's quadrature; the node
    counts of Table 1 are pinned in tests/test_workloads.py
  * targets: grid points outside the spheroid within distance h, 0 <= b <= h (PAPER.md:249,
    reading R13), x0 their closest points, n0 the outward normals there
  * single-layer density: f_1 = F0 / sqrt(1 - 3 x1^2 / 4), f_2 = f_3 = 0, the
    traction of the translating spheroid.  F0 = F / (2 pi) with the axial drag
    F = 6 pi a K, K = (8/3) e^3 / (-2e + (1 + e^2) ln((1+e)/(1-e))) (Oberbeck), a = 1,
    e = sqrt(3)/2 (the traction of a translating ellipsoid is F / (4 pi a b c |grad|) with
    |grad|^2 = x1^2/a^4 + x2^2/b^4 + x3^2/c^4, which is F / (2 pi sqrt(4 - 3 x1^2)) * 2 here)
  * rho = (3, 4, 5)

Inputs only; the exact velocity the errors are measured against is in tests/closed_forms.py.
"""
from __future__ import annotations

import math

import numpy as np

from .configs import Block, _c
from .quadrature import Ellipsoid, grid_targets_outside, quadrature

AXES = (1.0, 0.5, 0.5)          # PAPER.md:245 "x1^2 + 4 x2^2 + 4 x3^2 = 1"
RHO_SPHEROID = (3.0, 4.0, 5.0)  # PAPER.md:249 "rho = 3, 4, 5"
ECC = math.sqrt(1.0 - 0.25)     # e = sqrt(1 - (b/a)^2)
_LOG = math.log((1.0 + ECC) / (1.0 - ECC))
DRAG_K = (8.0 / 3.0) * ECC ** 3 / (-2.0 * ECC + (1.0 + ECC ** 2) * _LOG)
F0 = 6.0 * math.pi * DRAG_K / (2.0 * math.pi)


def traction(x):
    """f_1 = F0 / sqrt(1 - 3 x1^2 / 4), f_2 = f_3 = 0."""
    x = np.asarray(x, dtype=np.float64)
    f = np.zeros_like(x)
    f[0] = F0 / np.sqrt(1.0 - 0.75 * x[0] ** 2)
    return f


def spheroid_block(inv_h: int = 32) -> Block:
    """One SL evaluation of PAPER.md Table 1 at h = 1/inv_h (targets: grid points outside,
    within h).  q is zero (the benchmark is the Stokeslet integral alone)."""
    h = 1.0 / inv_h
    surf = Ellipsoid(AXES)
    x, n, w, _ = quadrature(surf, h)
    y, x0, b = grid_targets_outside(surf, h, h)
    g = x0 / (np.asarray(AXES)[:, None] ** 2)
    n0 = g / np.linalg.norm(g, axis=0, keepdims=True)
    f = traction(x)
    x0d = np.concatenate([n0, traction(x0), np.zeros_like(x0)], axis=0)
    return Block(_c(x), _c(n), _c(w), f, np.zeros_like(f), _c(y), _c(b), _c(x0d), h, RHO_SPHEROID,
                 f"spheroid_h1/{inv_h}", tgt_x0=_c(x0), meta={"config": "spheroid", "inv_h": inv_h})

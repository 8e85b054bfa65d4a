"""Seeded inputs of the two-drop interfacial Stokes flow (NEXT-2, Sec. 4.3).

Geometry and data only -- none of the layer-potential arithmetic lives here.

  * two unit spheres ("drops"), centres c_1 = (0, 0, 0) and c_2 = (2 + eps, 0, 0),
    eps = 1/16^3: SURVEY 8(c) reading 12 of PAPER.md:339 ("centered ... at (2,0,eps)",
    read as a typo for a centre separation 2 + eps along x_1; R17).  The
    literal (2, 0, eps) (gap sqrt(4 + eps^2) - 2 ~ 1.5e-8) is separation="z".  Each
    drop has its own centre-anchored quadrature grid;
  * viscosity ratios lambda_1 = lambda_2 = 2, mu_0 = 1;
  * interface force jump [f] = 2 gamma H n - grad_S gamma with gamma = 1 + (x_1 - x_c)^2,
    x_c the centre's x-coordinate, H = 1 (mean curvature of a unit sphere, the average of
    the principal curvatures) and n the outward normal (R18);
  * cross-block target data: the nodes of drop b seen from drop m != b, with the closest
    point x0 on sphere m (radial projection), b' = |y - c_m| - 1 > 0 (outside m) and
    [f]_m(x0) in closed form.

Self-convergence (eq. (36)) compares u_h and u_{h/2} at the coarse nodes:
the h-grid lines are h/2-grid lines, so every coarse node is a fine node
(`match_nodes`).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from .quadrature import quadrature, sphere

EPS_PAPER = 1.0 / 16 ** 3      # PAPER.md:339 "centered ... at (2,0,eps), where eps = 1/16^3"
LAMBDA_PAPER = 2.0             # PAPER.md:337 "lambda_1 = lambda_2 = 2"
RHO_TWODROP = (3.0, 4.0, 5.0)  # PAPER.md:341 "delta = {3h, 4h, 5h}" for the nearby-surface integrals
RHO_SELF = 3.0                 # PAPER.md:341 "delta = 3h" for the self-surface (on-surface) integrals
GMRES_TOL = 1e-10              # PAPER.md:343 "GMRES with a tolerance 10^{-10}"


def gamma(x, xc: float):
    """Surface tension gamma = 1 + (x_1 - x_c)^2."""
    return 1.0 + (x[0] - xc) ** 2


def jump_force(x, c):
    """[f] = 2 gamma H n - grad_S gamma on the unit sphere centred at c.

    x: (3, K) points on the sphere.  H = 1, n = x - c, grad gamma = (2 (x_1 - x_c), 0, 0),
    grad_S gamma = (I - n n^T) grad gamma."""
    x = np.asarray(x, dtype=np.float64)
    c = np.asarray(c, dtype=np.float64)[:, None]
    n = x - c
    n = n / np.linalg.norm(n, axis=0, keepdims=True)
    g = gamma(x, float(c[0, 0]))
    grad = np.zeros_like(x)
    grad[0] = 2.0 * (x[0] - c[0, 0])
    grad_s = grad - (n * grad).sum(axis=0, keepdims=True) * n
    return np.ascontiguousarray(2.0 * g * 1.0 * n - grad_s)


@dataclass
class Drop:
    center: np.ndarray  # (3,)
    x: np.ndarray       # (3, N) nodes
    n: np.ndarray       # (3, N) outward unit normals
    w: np.ndarray       # (N,)   quadrature weights
    f: np.ndarray       # (3, N) [f] at the nodes
    lam: float          # viscosity ratio mu_m / mu_0

    @property
    def N(self) -> int:
        return int(self.x.shape[1])


@dataclass
class Cross:
    """Targets = nodes of drop `tgt`, sources = drop `src` != tgt."""
    tgt: int
    src: int
    b: np.ndarray       # (N_tgt,) signed distance to sphere src (> 0: outside it)
    x0: np.ndarray      # (3, N_tgt) closest point on sphere src
    n0: np.ndarray      # (3, N_tgt) outward normal of sphere src at x0
    f0: np.ndarray      # (3, N_tgt) [f]_src(x0)


@dataclass
class TwoDrop:
    h: float
    drops: list
    cross: list                     # cross[b] = Cross(tgt=b, src=1-b)
    rho: tuple = RHO_TWODROP
    delta_self: float = 0.0
    tol: float = GMRES_TOL
    meta: dict = field(default_factory=dict)

    @property
    def n_unknowns(self) -> int:
        return 3 * sum(d.N for d in self.drops)


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def twodrop(inv_h: int = 16, eps: float = EPS_PAPER, lam=(LAMBDA_PAPER, LAMBDA_PAPER),
            separation: str = "x") -> TwoDrop:
    """The PAPER.md Sec. 4.3 two-drop inputs at grid spacing h = 1/inv_h.

    separation "x" (default, R17): c_2 = (2 + eps, 0, 0), a gap eps along x_1;
    "z": c_2 = (2, 0, eps), PAPER.md:339 taken literally."""
    h = 1.0 / inv_h
    c1 = np.zeros(3)
    c2 = np.array([2.0, 0.0, eps]) if separation == "z" else np.array([2.0 + eps, 0.0, 0.0])
    drops = []
    for c, lm in ((c1, lam[0]), (c2, lam[1])):
        x, n, w, _ = quadrature(sphere(1.0, tuple(c)), h)
        drops.append(Drop(c.copy(), _c(x), _c(n), _c(w), jump_force(x, c), float(lm)))
    cross = []
    for b in range(2):
        m = 1 - b
        rel = drops[b].x - drops[m].center[:, None]
        R = np.linalg.norm(rel, axis=0)
        n0 = rel / R
        x0 = drops[m].center[:, None] + n0
        cross.append(Cross(b, m, _c(R - 1.0), _c(x0), _c(n0), jump_force(x0, drops[m].center)))
    return TwoDrop(h, drops, cross, RHO_TWODROP, RHO_SELF * h, GMRES_TOL,
                   meta={"inv_h": inv_h, "eps": eps, "separation": separation,
                         "lambda": tuple(float(v) for v in lam)})


def match_nodes(coarse: TwoDrop, fine: TwoDrop, tol: float = 1e-10):
    """Index of every coarse node among the fine nodes, per drop (grid nesting, eq. (36))."""
    from scipy.spatial import cKDTree

    out = []
    for dc, df in zip(coarse.drops, fine.drops):
        dist, idx = cKDTree(df.x.T).query(dc.x.T)
        if not np.all(dist <= tol):
            raise ValueError(f"coarse node without a fine counterpart (max dist {dist.max():.3g})")
        out.append(idx)
    return out


def split(td: TwoDrop, vec):
    """Stacked unknown vector (3*(N_1+N_2),) -> [u_1 (3,N_1), u_2 (3,N_2)] (SoA per drop)."""
    vec = np.asarray(vec)
    n1 = td.drops[0].N
    return [vec[:3 * n1].reshape(3, n1), vec[3 * n1:].reshape(3, td.drops[1].N)]


def stack(parts):
    return np.concatenate([np.ascontiguousarray(p).reshape(-1) for p in parts])

"""Seeded input generation, part 1: surfaces and the projection quadrature.

This module builds INPUTS shared by the CUDA path's tests/bench and by the
CPU oracle.  It holds none of the hot path's arithmetic (no kernels, no
s-factors, no extrapolation); it only produces quadrature nodes x, unit
normals n(x) and weights w(x) on analytic quadrics.

Quadrature rule: PAPER.md Sec. 2.2 "Quadrature", lines 142-160, eq. (23)
(`quadrature`) and the partition of unity of lines 151-159:

  * Gamma_i = points x whose two coordinates other than x_i are grid values
    (multiples of h, grid anchored at the surface centre) and whose normal
    satisfies |n(x).e_i| >= cos(theta), theta = 70 degrees
  * w_i(x) = psi_i(n(x)) / |n_i(x)| * h^2
  * bump b(r) = exp(2 r^2/(r^2-1)) for |r|<1, else 0
  * beta_i(n) = b(arccos|n_i| / theta), psi_i = beta_i / sum_j beta_j
    (the source's parenthesis is garbled, R10)

The grid is anchored at the quadric's centre; both roots of every grid line
are kept.  With this reading the node counts of PAPER.md Table 1 (lines
266-272) are reproduced exactly (tests/test_workloads.py).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

THETA_Q = math.radians(70.0)  # PAPER.md:145 "we take theta = 70 deg"


def bump(r):
    """b(r) = exp(2r^2/(r^2-1)) for |r| < 1, else 0."""
    r = np.asarray(r, dtype=np.float64)
    out = np.zeros_like(r)
    m = np.abs(r) < 1.0
    rr = r[m] * r[m]
    out[m] = np.exp(2.0 * rr / (rr - 1.0))
    return out


def partition_of_unity(n):
    """psi_i(n) = beta_i / sum_j beta_j, beta_i = b(arccos|n_i|/theta).

    n: (3, K) unit normals.  Returns psi (3, K)."""
    n = np.asarray(n, dtype=np.float64)
    ang = np.arccos(np.clip(np.abs(n), 0.0, 1.0))
    beta = bump(ang / THETA_Q)
    return beta / beta.sum(axis=0, keepdims=True)


@dataclass(frozen=True)
class Ellipsoid:
    """Quadric sum_i ((x_i - c_i)/a_i)^2 = 1; a sphere when a1 = a2 = a3."""

    axes: tuple = (1.0, 1.0, 1.0)
    center: tuple = (0.0, 0.0, 0.0)

    def level(self, x):
        a = np.asarray(self.axes)[:, None]
        c = np.asarray(self.center)[:, None]
        return (((x - c) / a) ** 2).sum(axis=0) - 1.0

    def normal(self, x):
        a = np.asarray(self.axes)[:, None]
        c = np.asarray(self.center)[:, None]
        g = (x - c) / (a * a)
        return g / np.linalg.norm(g, axis=0, keepdims=True)


def sphere(radius=1.0, center=(0.0, 0.0, 0.0)) -> Ellipsoid:
    return Ellipsoid((radius, radius, radius), tuple(center))


def quadrature(surface: Ellipsoid, h: float):
    """Projection quadrature of PAPER.md Sec. 2.2 on an ellipsoid.

    Returns (x (3,N), n (3,N), w (N,), set_index (N,) in {0,1,2}).
    Nodes are ordered set by set (Gamma_1, Gamma_2, Gamma_3), each by grid line.
    """
    a = np.asarray(surface.axes, dtype=np.float64)
    c = np.asarray(surface.center, dtype=np.float64)
    cos_t = math.cos(THETA_Q)
    xs, ns, ws, ids = [], [], [], []
    for i in range(3):
        j, k = [d for d in range(3) if d != i]
        mj = int(math.floor(a[j] / h))
        mk = int(math.floor(a[k] / h))
        gj = np.arange(-mj, mj + 1, dtype=np.float64) * h
        gk = np.arange(-mk, mk + 1, dtype=np.float64) * h
        GJ, GK = np.meshgrid(gj, gk, indexing="ij")
        GJ = GJ.ravel()
        GK = GK.ravel()
        s = 1.0 - (GJ / a[j]) ** 2 - (GK / a[k]) ** 2
        keep = s > 0.0
        GJ, GK, s = GJ[keep], GK[keep], s[keep]
        root = a[i] * np.sqrt(s)
        for sign in (1.0, -1.0):
            p = np.empty((3, GJ.size))
            p[i] = sign * root
            p[j] = GJ
            p[k] = GK
            g = p / (a[:, None] ** 2)
            nrm = g / np.linalg.norm(g, axis=0, keepdims=True)
            sel = np.abs(nrm[i]) >= cos_t
            p = p[:, sel]
            nrm = nrm[:, sel]
            psi = partition_of_unity(nrm)
            w = psi[i] / np.abs(nrm[i]) * h * h
            xs.append(p + c[:, None])
            ns.append(nrm)
            ws.append(w)
            ids.append(np.full(p.shape[1], i, dtype=np.int32))
    x = np.ascontiguousarray(np.concatenate(xs, axis=1))
    n = np.ascontiguousarray(np.concatenate(ns, axis=1))
    w = np.ascontiguousarray(np.concatenate(ws))
    return x, n, w, np.concatenate(ids)


def ellipsoid_closest_point(surface: Ellipsoid, y, iters: int = 200):
    """Closest point on an ellipsoid by bisection on the Lagrange multiplier.

    For y outside (or on) the ellipsoid, x_i = a_i^2 y_i / (a_i^2 + t) with t >= 0
    the root of F(t) = sum (a_i y_i / (a_i^2 + t))^2 - 1.  Used only to
    classify grid targets for the Table-1 count pin.
    y: (3, K) points with level >= 0.  Returns (x0 (3,K), dist (K,)).
    """
    a = np.asarray(surface.axes, dtype=np.float64)[:, None]
    c = np.asarray(surface.center, dtype=np.float64)[:, None]
    yy = np.asarray(y, dtype=np.float64) - c
    lo = np.zeros(yy.shape[1])
    hi = np.linalg.norm(yy, axis=0) * a.max() + 1e-300
    for _ in range(iters):
        mid = 0.5 * (lo + hi)
        F = ((a * yy / (a * a + mid)) ** 2).sum(axis=0) - 1.0
        pos = F > 0.0
        lo = np.where(pos, mid, lo)
        hi = np.where(pos, hi, mid)
    t = 0.5 * (lo + hi)
    x0 = a * a * yy / (a * a + t)
    return x0 + c, np.linalg.norm(yy - x0, axis=0)


def grid_targets_outside(surface: Ellipsoid, h: float, dist_max: float):
    """3-D grid points y = (i h, j h, k h) on or outside the surface with distance
    0 <= b <= dist_max ("grid points outside ... within distance h").
    Returns (y (3,M), x0 (3,M), b (M,))."""
    a = np.asarray(surface.axes)
    c = np.asarray(surface.center)
    rng = [np.arange(math.floor((c[d] - a[d] - dist_max) / h) - 1,
                     math.ceil((c[d] + a[d] + dist_max) / h) + 2) * h for d in range(3)]
    G = np.stack(np.meshgrid(*rng, indexing="ij")).reshape(3, -1)
    lev = surface.level(G)
    # cheap prefilter on the level function before the exact distance
    a_min = a.min()
    shell = (lev >= 0.0) & (lev <= (1.0 + dist_max / a_min) ** 2 - 1.0 + 1e-12)
    G = G[:, shell]
    x0, dist = ellipsoid_closest_point(surface, G)
    on = surface.level(G) == 0.0
    dist = np.where(on, 0.0, dist)
    # b = dist_max exactly (e.g. grid points on the symmetry axes) must survive rounding
    keep = dist <= dist_max * (1.0 + 1e-9)
    return G[:, keep], x0[:, keep], dist[keep]

"""Seeded synthetic workloads for BASELINE.json configs 1-5 (recipe: DESIGN.md Sec. 3).

A `Block` is exactly the argument set of one `stokes_er_eval` call
(include/stokes_er.h): one source surface, one target set whose (b, x0, n0)
are relative to that surface, densities at the nodes and at x0.  All arrays
are float64, C-contiguous, SoA [rows][count].

Every random draw comes from numpy PCG64 seeded with the config index unless
a seed is passed.  Nothing here computes any part of the layer potentials.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, replace

import numpy as np

from .densities import Field, PolyField, TrigField
from .quadrature import Ellipsoid, quadrature, sphere

RHO_CONFIGS = (2.0, 3.0, 4.0)  # BASELINE.json configs: rho = (2,3,4)


@dataclass
class Block:
    src_xyz: np.ndarray         # (3, N) quadrature nodes x
    src_normal: np.ndarray      # (3, N) unit outward normals n(x)
    src_weight: np.ndarray      # (N,)   quadrature weights w(x) > 0
    f: np.ndarray               # (3, N) single-layer density at the nodes
    q: np.ndarray               # (3, N) double-layer density at the nodes
    tgt_xyz: np.ndarray         # (3, M) targets y
    tgt_b: np.ndarray           # (M,)   signed distance, > 0 outside
    tgt_x0_density: np.ndarray  # (9, M) rows: n0(3), f(x0)(3), q(x0)(3)
    h: float
    rho: tuple = RHO_CONFIGS
    name: str = ""
    tgt_x0: np.ndarray | None = None      # (3, M) closest points (for closed-form checks only)
    meta: dict = field(default_factory=dict)

    @property
    def N(self) -> int:
        return int(self.src_xyz.shape[1])

    @property
    def M(self) -> int:
        return int(self.tgt_xyz.shape[1])

    def arrays(self):
        return (self.src_xyz, self.src_normal, self.src_weight, self.f, self.q,
                self.tgt_xyz, self.tgt_b, self.tgt_x0_density)

    def input_bytes(self) -> int:
        return sum(a.nbytes for a in self.arrays())

    def take_targets(self, idx) -> "Block":
        idx = np.asarray(idx)
        c = lambda a: np.ascontiguousarray(a[..., idx])
        return replace(self, tgt_xyz=c(self.tgt_xyz), tgt_b=c(self.tgt_b),
                       tgt_x0_density=c(self.tgt_x0_density),
                       tgt_x0=None if self.tgt_x0 is None else c(self.tgt_x0),
                       meta=dict(self.meta, target_subsample=len(idx)))


def _c(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def make_block(surface: Ellipsoid, h: float, y, b, x0, n0, f_field: Field, q_field: Field,
               rho=RHO_CONFIGS, name="", src=None, meta=None) -> Block:
    """Assemble a Block: nodes from the quadrature of `surface` (or `src`), densities
    from the analytic fields, x0-densities from the same fields at x0."""
    if src is None:
        x, n, w, _ = quadrature(surface, h)
    else:
        x, n, w = src
    dens = np.concatenate([n0, f_field(x0), q_field(x0)], axis=0)
    return Block(_c(x), _c(n), _c(w), _c(f_field(x)), _c(q_field(x)), _c(y), _c(b), _c(dens),
                 float(h), tuple(float(r) for r in rho), name, tgt_x0=_c(x0), meta=dict(meta or {}))


def random_directions(rng: np.random.Generator, m: int):
    d = rng.standard_normal((3, m))
    return d / np.linalg.norm(d, axis=0, keepdims=True)


def sphere_shell_targets(rng, m, bmin, bmax=None, center=(0.0, 0.0, 0.0), radius=1.0, b_values=None):
    """Targets y = x0 + b n0 around a sphere; x0 = c + R d for random unit d."""
    d = random_directions(rng, m)
    b = np.asarray(b_values, dtype=np.float64) if b_values is not None else rng.uniform(bmin, bmax, m)
    c = np.asarray(center, dtype=np.float64)[:, None]
    x0 = c + radius * d
    return x0 + b * d, b, x0, d


def config1(seed: int = 1, f_field: Field | None = None, q_field: Field | None = None,
            per_class: int = 72, inv_h: int = 16, rho=RHO_CONFIGS) -> Block:
    """Config 1: unit sphere, 1/h = 16; per_class targets for each b/h in {0,+-1,+-2,+-3}."""
    rng = np.random.default_rng(seed)
    h = 1.0 / inv_h
    classes = np.repeat(np.array([0, 1, -1, 2, -2, 3, -3], dtype=np.float64), per_class) * h
    y, b, x0, n0 = sphere_shell_targets(rng, classes.size, None, b_values=classes)
    f_field = f_field or PolyField(rng)
    q_field = q_field or PolyField(rng)
    return make_block(sphere(), h, y, b, x0, n0, f_field, q_field, rho, name=f"cfg1_sphere_h1/{inv_h}",
                      meta={"config": 1, "seed": seed})


def config2(inv_h: int = 64, seed: int = 2, f_field=None, q_field=None, rho=RHO_CONFIGS) -> Block:
    """Config 2: unit sphere; all N nodes as targets (b = 0) + N/2 shell targets, b ~ U[-3h, 3h]."""
    rng = np.random.default_rng(seed)
    h = 1.0 / inv_h
    x, n, w, _ = quadrature(sphere(), h)
    N = x.shape[1]
    ys, bs, x0s, n0s = sphere_shell_targets(rng, N // 2, -3 * h, 3 * h)
    y = np.concatenate([x, ys], axis=1)
    b = np.concatenate([np.zeros(N), bs])
    x0 = np.concatenate([x, x0s], axis=1)
    n0 = np.concatenate([n, n0s], axis=1)
    f_field = f_field or PolyField(rng)
    q_field = q_field or PolyField(rng)
    return make_block(sphere(), h, y, b, x0, n0, f_field, q_field, rho, name=f"cfg2_sphere_h1/{inv_h}",
                      src=(x, n, w), meta={"config": 2, "seed": seed})


def config3(inv_h: int = 64, seed: int = 3, rho=RHO_CONFIGS) -> Block:
    """Config 3: ellipsoid (1, 0.8, 0.6); all nodes (b = 0) + N/2 near points
    y = x0 + b n0, x0 a random node, b ~ U[-2h, 2h] (|b| << min curvature radius 0.36)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / inv_h
    surf = Ellipsoid((1.0, 0.8, 0.6))
    x, n, w, _ = quadrature(surf, h)
    N = x.shape[1]
    pick = rng.integers(0, N, N // 2)
    bs = rng.uniform(-2 * h, 2 * h, N // 2)
    x0s, n0s = x[:, pick], n[:, pick]
    y = np.concatenate([x, x0s + bs * n0s], axis=1)
    b = np.concatenate([np.zeros(N), bs])
    x0 = np.concatenate([x, x0s], axis=1)
    n0 = np.concatenate([n, n0s], axis=1)
    f_field = TrigField(rng)
    q_field = TrigField(rng)
    return make_block(surf, h, y, b, x0, n0, f_field, q_field, rho, name=f"cfg3_ellipsoid_h1/{inv_h}",
                      src=(x, n, w), meta={"config": 3, "seed": seed})


def config4(eps: float = 0.1, inv_h: int = 64, seed: int = 4, rho=RHO_CONFIGS, f_field=None, q_field=None):
    """Config 4: two unit spheres, centres 0 and (2+eps, 0, 0), each with its own
    centre-anchored grid.  Returns the 4 blocks [A<-A, A<-B, B<-A, B<-B]
    (targets <- sources); a cross block's (b, x0, n0) are relative to the
    source sphere (R12)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / inv_h
    cA = np.zeros(3)
    cB = np.array([2.0 + eps, 0.0, 0.0])
    xA, nA, wA, _ = quadrature(sphere(1.0, cA), h)
    xB, nB, wB, _ = quadrature(sphere(1.0, cB), h)
    f_field = f_field or PolyField(rng)
    q_field = q_field or PolyField(rng)
    nodes = {"A": (xA, nA, wA, cA), "B": (xB, nB, wB, cB)}
    blocks = []
    for tname in "AB":
        for sname in "AB":
            xt, nt, _, _ = nodes[tname]
            xs, ns, ws, cs = nodes[sname]
            if tname == sname:
                y, b, x0, n0 = xt, np.zeros(xt.shape[1]), xt, nt
            else:
                rel = xt - cs[:, None]
                R = np.linalg.norm(rel, axis=0)
                n0 = rel / R
                x0 = cs[:, None] + n0
                b = R - 1.0
                y = xt
            blocks.append(make_block(None, h, y, b, x0, n0, f_field, q_field, rho,
                                     name=f"cfg4_eps{eps}_{tname}<-{sname}", src=(xs, ns, ws),
                                     meta={"config": 4, "seed": seed, "eps": eps}))
    return blocks


def config5(inv_h: int = 128, seed: int = 5, rho=RHO_CONFIGS) -> Block:
    """Config 5: unit sphere, M = N on-surface node targets (b = 0)."""
    rng = np.random.default_rng(seed)
    h = 1.0 / inv_h
    x, n, w, _ = quadrature(sphere(), h)
    f_field = PolyField(rng)
    q_field = PolyField(rng)
    return make_block(sphere(), h, x, np.zeros(x.shape[1]), x, n, f_field, q_field, rho,
                      name=f"cfg5_sphere_h1/{inv_h}", src=(x, n, w), meta={"config": 5, "seed": seed})


def node_block(block: Block, name_suffix: str = "_nodes") -> Block:
    """The Block whose targets are `block`'s own quadrature nodes: y = x, b = 0, x0 = x,
    n0 = n, f(x0) = f and q(x0) = q at the node -- the argument set of stokes_er_eval that
    stokes_er_eval_nodes computes (include/stokes_er.h)."""
    x = block.src_xyz
    dens = np.concatenate([block.src_normal, block.f, block.q], axis=0)
    return replace(block, tgt_xyz=_c(x), tgt_b=np.zeros(x.shape[1]), tgt_x0_density=_c(dens), tgt_x0=_c(x),
                   name=block.name + name_suffix, meta=dict(block.meta, targets="nodes"))


def pure_far(inv_h: int = 128, seed: int = 6, b: float = 0.5, rho=RHO_CONFIGS) -> Block:
    """Far-only micro-workload: sphere nodes as sources, M = N targets at b = 0.5.
    Every pair has r >= 0.5 > 6*delta_max for 1/h >= 64."""
    rng = np.random.default_rng(seed)
    h = 1.0 / inv_h
    x, n, w, _ = quadrature(sphere(), h)
    y = (1.0 + b) * n
    f_field = PolyField(rng)
    q_field = PolyField(rng)
    return make_block(sphere(), h, y, np.full(x.shape[1], b), n.copy(), n, f_field, q_field, rho,
                      name=f"pure_far_h1/{inv_h}", src=(x, n, w), meta={"config": "far", "seed": seed})


def make_config(idx: int, **kw):
    return {1: config1, 2: config2, 3: config3, 4: config4, 5: config5}[idx](**kw)


def subsample(block: Block, k: int, seed: int = 12345) -> Block:
    """Seeded target subsample for oracle parity at large M:
    always keeps the first and last target plus k-2 random ones, sorted."""
    if block.M <= k:
        return block
    rng = np.random.default_rng(seed)
    idx = np.unique(np.concatenate([[0, block.M - 1], rng.choice(block.M, k - 2, replace=False)]))
    return block.take_targets(idx)

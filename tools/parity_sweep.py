#!/usr/bin/env python
"""Randomized parity sweep of the CUDA path against the oracle (run on the GPU box).

Each case draws a seeded random geometry (sphere or ellipsoid, random semi-axes and centre),
h in {1/8, 1/12, 1/16, 1/24}, a strictly increasing rho triple in [1.5, 6], a mode (SL, DL, both),
densities (polynomial or trigonometric) and a target mix (nodes with b = 0, a shell with
b ~ U[-4h, 4h], a few far targets), then compares stokes_er_eval with the oracle's localized
mode (max-norm relative, u and v separately; the bar is 1e-12).  Every fifth case also runs
the on-surface s# variant (random delta in [2h, 4h], cutoff 7) on the node targets, and every
fourth the treecode (random N0 in [40, 600), p in [2, 8], theta in [0.3, 0.8]) against the
treecode oracle, and every third the node-target path (stokes_er_eval_nodes) on all the nodes.

    python tools/parity_sweep.py OUT.json [n_cases]
"""
from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import oracle  # noqa: E402  (test infrastructure: this is a parity check)
import paper_2507_00156_b200 as ser  # noqa: E402
from workloads.configs import make_block, node_block, random_directions  # noqa: E402
from workloads.densities import PolyField, TrigField  # noqa: E402
from workloads.quadrature import Ellipsoid, ellipsoid_closest_point, quadrature  # noqa: E402


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def case(seed: int):
    rng = np.random.default_rng(10_000 + seed)
    axes = (1.0, 1.0, 1.0) if rng.random() < 0.5 else tuple(np.sort(rng.uniform(0.6, 1.2, 3))[::-1])
    center = tuple(rng.uniform(-0.5, 0.5, 3))
    surf = Ellipsoid(axes, center)
    inv_h = int(rng.choice([8, 12, 16, 24]))
    h = 1.0 / inv_h
    rho = tuple(np.sort(rng.choice(np.arange(1.5, 6.01, 0.25), 3, replace=False)))
    mode = int(rng.choice([1, 2, 3]))
    x, n, w, _ = quadrature(surf, h)
    N = x.shape[1]
    k_nodes = min(N, int(rng.integers(20, 400)))
    pick = rng.choice(N, k_nodes, replace=False)
    m_shell = int(rng.integers(50, 500))
    # shell targets: a random node as x0, b ~ U[-4h, 4h] along its normal (|b| << curvature radii)
    sp = rng.integers(0, N, m_shell)
    bs = rng.uniform(-4 * h, 4 * h, m_shell)
    m_far = int(rng.integers(0, 8))
    d = random_directions(rng, m_far)
    yf = np.asarray(center)[:, None] + 8.0 * d  # beyond 6 delta_max of every node: no near pairs, w = (1,0,0)
    x0f, bf = ellipsoid_closest_point(surf, yf)
    n0f = surf.normal(x0f)
    y = np.concatenate([x[:, pick], x[:, sp] + bs * n[:, sp], yf], axis=1)
    b = np.concatenate([np.zeros(k_nodes), bs, bf])
    x0 = np.concatenate([x[:, pick], x[:, sp], x0f], axis=1)
    n0 = np.concatenate([n[:, pick], n[:, sp], n0f], axis=1)
    fields = (PolyField(rng), PolyField(rng)) if rng.random() < 0.5 else (TrigField(rng), TrigField(rng))
    blk = make_block(surf, h, y, b, x0, n0, *fields, rho=rho, name=f"sweep{seed}", src=(x, n, w))
    return blk, mode, k_nodes


def main(out, n_cases=60):
    rows = []
    t0 = time.time()
    for seed in range(n_cases):
        blk, mode, k_nodes = case(seed)
        u, v = ser.evaluate_block(blk, mode=mode)
        ur, vr = oracle.evaluate_block(blk, mode=mode, localized=True)
        row = {"seed": seed, "N": blk.N, "M": blk.M, "inv_h": round(1 / blk.h), "rho": blk.rho, "mode": mode}
        if mode & 1:
            row["rel_u"] = rel(u.cpu().numpy(), ur)
        if mode & 2:
            row["rel_v"] = rel(v.cpu().numpy(), vr)
        if seed % 5 == 0:  # NEXT-1 on the node targets
            sub = blk.take_targets(np.arange(k_nodes))
            delta = float(np.random.default_rng(seed).uniform(2, 4)) * blk.h
            us, vs = ser.evaluate_onsurface(*ser.to_device(sub), delta, mode=mode)
            usr, vsr = oracle.evaluate_sharp(*sub.arrays(), delta, mode=mode, localized=True, cutoff=7.0)
            if mode & 1:
                row["sharp_rel_u"] = rel(us.cpu().numpy(), usr)
            if mode & 2:
                row["sharp_rel_v"] = rel(vs.cpu().numpy(), vsr)
        if seed % 4 == 1:  # NEXT-3: random treecode parameters against the treecode oracle
            trng = np.random.default_rng(50_000 + seed)
            n0, deg, th = int(trng.integers(40, 600)), int(trng.integers(2, 9)), float(trng.uniform(0.3, 0.8))
            ut, vt = ser.evaluate_tree_block(blk, mode=mode, leaf_size=n0, degree=deg, theta=th)
            utr, vtr = oracle.evaluate_tree_block(blk, mode=mode, leaf_size=n0, degree=deg, theta=th)
            row["tree"] = [n0, deg, th]
            if mode & 1:
                row["tree_rel_u"] = rel(ut.cpu().numpy(), utr)
            if mode & 2:
                row["tree_rel_v"] = rel(vt.cpu().numpy(), vtr)
        if seed % 3 == 2:  # node targets: stokes_er_eval_nodes (symmetric far kernel) on every node
            nb = node_block(blk)
            un, vn = ser.evaluate_nodes_block(nb, mode=mode)
            unr, vnr = oracle.evaluate_block(nb, mode=mode, localized=True)
            if mode & 1:
                row["nodes_rel_u"] = rel(un.cpu().numpy(), unr)
            if mode & 2:
                row["nodes_rel_v"] = rel(vn.cpu().numpy(), vnr)
        rows.append(row)
        print(row, flush=True)
    worst = max(v for r in rows for k, v in r.items() if k.startswith(("rel_", "sharp_rel_", "tree_rel_", "nodes_rel_")))
    res = {"what": "randomized parity sweep: stokes_er_eval (every 5th case also stokes_er_eval_onsurface, every "
                   "4th also stokes_er_eval_tree with random N0, p, theta, every 3rd also stokes_er_eval_nodes on "
                   "all nodes) vs the oracle's localized mode (treecode: vs the treecode oracle), max-norm "
                   "relative per output",
           "cases": len(rows), "worst_rel": worst, "bar": 1e-12, "pass": bool(worst <= 1e-12),
           "seconds": time.time() - t0, "rows": rows}
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "rows"}))
    return 0 if res["pass"] else 1


if __name__ == "__main__":
    sys.exit(main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 60))

#!/usr/bin/env python
"""PAPER.md Fig. 6 (direct O(N^2) vs treecode O(N log N)) and Sec. 4.2's parameter
policy on one B200: config 5 (unit sphere, M = N on-surface targets) at
1/h = 32 ... 256; for each h the direct stokes_er_eval and stokes_er_eval_tree
with theta = 0.6, N0 = 2000 * 2^k, p = 6 + 2k at h = 1/64 / 2^k (eq. (33)),
device time per evaluation (CUDA events, median of reps), and the treecode's
max-norm relative difference from the direct sum.  Optional extra (N0, p)
pairs per h probe the trade-off.

    python tools/tree_scaling.py out.json [inv_h ...]
"""
import json
import os
import statistics
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import paper_2507_00156_b200 as ser  # noqa: E402
from workloads.configs import config5  # noqa: E402


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts)


def policy(inv_h):
    k = int(round(np.log2(inv_h / 64)))
    return int(2000 * 2.0 ** k), 6 + 2 * k


out = sys.argv[1] if len(sys.argv) > 1 else None
levels = [int(a) for a in sys.argv[2:]] or [32, 64, 128, 256]
rows = []
for ih in levels:
    blk = config5(inv_h=ih)
    arrs = ser.to_device(blk)
    M, N = blk.M, blk.N
    u = torch.empty((3, M), dtype=torch.float64, device="cuda")
    v = torch.empty((3, M), dtype=torch.float64, device="cuda")
    ws = ser.alloc_workspace(M, N)
    reps = 5 if N < 300000 else 2
    t_dir = timed(lambda: ser.evaluate(*arrs, blk.h, blk.rho, out_u=u, out_v=v, workspace=ws), reps)
    ud, vd = u.clone(), v.clone()
    N0, p = policy(ih)
    cands = [(N0, p, 0.6)]
    if ih >= 64:
        cands += [(N0 // 2, p, 0.6), (N0, p - 2, 0.6), (N0, p + 2, 0.6)]
    for (n0, pp, th) in cands:
        if pp < 2 or n0 < 64:
            continue
        t0 = time.perf_counter()
        plan = ser.TreePlan(blk.src_xyz, n0, pp, th)
        t_build = time.perf_counter() - t0
        nbytes = int(ser._lib.load().stokes_er_tree_workspace_bytes(M, N, 3, __import__("ctypes").byref(plan.params),
                                                                      plan.ptr()))
        tws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        ut = torch.empty_like(u)
        vt = torch.empty_like(v)
        t_tree = timed(lambda: ser.evaluate_tree(*arrs, blk.h, blk.rho, plan, out_u=ut, out_v=vt, workspace=tws), reps)
        eu = float((ut - ud).abs().max() / ud.abs().max())
        ev = float((vt - vd).abs().max() / vd.abs().max())
        row = {"inv_h": ih, "N": N, "M": M, "direct_ms": t_dir, "N0": n0, "p": pp, "theta": th, "tree_ms": t_tree,
               "speedup": t_dir / t_tree, "nodes": plan.nodes, "depth": plan.depth, "host_build_s": t_build,
               "rel_diff_u": eu, "rel_diff_v": ev, "policy": (n0, pp) == (N0, p)}
        rows.append(row)
        print(row, flush=True)
res = {"what": "config 5 (unit sphere, M = N), direct vs treecode (PAPER.md Sec. 3.4, eq. (33) policy), one B200",
       "gpu": torch.cuda.get_device_name(), "rows": rows}
if out:
    json.dump(res, open(out, "w"), indent=1)

#!/usr/bin/env python
"""PAPER.md Sec. 4.2 (lines 276-318) on one B200: the treecode on the spheroid benchmark
(Table 1's SL evaluation) -- L2 error against the exact velocity and device time for
theta in {0.4, 0.6, 0.8}, p in {6, 8, 10, 12}, N0 in {2000, 4000, 8000} at 1/h = 128, and
the eq. (33) policy at 1/h = 64 ... 256, next to the direct sum.

    python tools/spheroid_tree.py out.json
"""
import ctypes
import json
import os
import statistics
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import torch  # noqa: E402

import paper_2507_00156_b200 as ser  # noqa: E402
from closed_forms import spheroid_translation_velocity  # noqa: E402
from workloads.spheroid import spheroid_block  # noqa: E402


def timed(fn, reps=3):
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


rows = []
cases = [(128, n0, p, th) for th in (0.4, 0.6, 0.8) for p in (6, 8, 10, 12) for n0 in (2000, 4000, 8000)]
cases += [(64, 2000, 6, 0.6), (256, 8000, 10, 0.6), (256, 8000, 8, 0.6)]
blocks = {}
for ih, n0, p, th in cases:
    if ih not in blocks:
        blk = spheroid_block(ih)
        arrs = ser.to_device(blk)
        ex = spheroid_translation_velocity(blk.tgt_xyz)
        u = torch.empty((3, blk.M), dtype=torch.float64, device="cuda")
        t_dir = timed(lambda: ser.evaluate(*arrs, blk.h, blk.rho, mode=1, out_u=u))
        e = np.linalg.norm(u.cpu().numpy() - ex, axis=0)
        blocks[ih] = (blk, arrs, ex, t_dir, float(np.sqrt((e ** 2).mean())), float(e.max()))
    blk, arrs, ex, t_dir, l2_dir, mx_dir = blocks[ih]
    plan = ser.TreePlan(blk.src_xyz, n0, p, th)
    nb = int(ser._lib.load().stokes_er_tree_workspace_bytes(blk.M, blk.N, 1, ctypes.byref(plan.params), plan.ptr()))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    ut = torch.empty((3, blk.M), dtype=torch.float64, device="cuda")
    t = timed(lambda: ser.evaluate_tree(*arrs, blk.h, blk.rho, plan, mode=1, out_u=ut, workspace=ws))
    e = np.linalg.norm(ut.cpu().numpy() - ex, axis=0)
    row = {"inv_h": ih, "N0": n0, "p": p, "theta": th, "tree_ms": t, "direct_ms": t_dir,
           "l2_err": float(np.sqrt((e ** 2).mean())), "max_err": float(e.max()), "direct_l2_err": l2_dir,
           "direct_max_err": mx_dir}
    rows.append(row)
    print(row, flush=True)
out = {"what": "treecode on PAPER.md Table 1's spheroid SL evaluation (Sec. 4.2), one B200", "rows": rows}
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)

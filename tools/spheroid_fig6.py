#!/usr/bin/env python
"""PAPER.md Fig. 6 (lines 318-327: CPU time vs N, direct O(N^2) vs treecode O(N log N)) as measured on
one B200 for the paper's own workload (the Table 1 spheroid SL evaluation): direct and treecode
(eq. (33) policy: theta 0.6; N0 2000, p 6 at h = 1/64; N0 x 2, p + 2 per halving) device times and
L2 errors against the exact velocity at 1/h = 32 ... 256.

    python tools/spheroid_fig6.py out.json
"""
import ctypes
import json
import math
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

PAPER_DIRECT_4THREADS_S = {32: 1.0, 64: 11.0, 128: 155.0, 256: 2461.0}  # PAPER.md Table 1


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
for ih in (32, 64, 128, 256):
    blk = spheroid_block(ih)
    arrs = ser.to_device(blk)
    ex = spheroid_translation_velocity(blk.tgt_xyz)
    u = torch.empty((3, blk.M), dtype=torch.float64, device="cuda")
    t_dir = timed(lambda: ser.evaluate(*arrs, blk.h, blk.rho, mode=1, out_u=u))
    e_dir = np.linalg.norm(u.cpu().numpy() - ex, axis=0)
    k = int(round(math.log2(ih / 64)))
    n0, p = int(2000 * 2.0 ** k), max(2, 6 + 2 * k)
    plan = ser.TreePlan(blk.src_xyz, n0, p, 0.6)
    nb = int(ser._lib.load().stokes_er_tree_workspace_bytes(blk.M, blk.N, 1, ctypes.byref(plan.params), plan.ptr()))
    ws = torch.empty(nb, dtype=torch.uint8, device="cuda")
    t_tree = timed(lambda: ser.evaluate_tree(*arrs, blk.h, blk.rho, plan, mode=1, out_u=u, workspace=ws))
    e_tree = np.linalg.norm(u.cpu().numpy() - ex, axis=0)
    row = {"inv_h": ih, "N": blk.N, "M": blk.M, "direct_ms": t_dir, "tree_ms": t_tree, "N0": n0, "p": p,
           "direct_l2": float(np.sqrt((e_dir ** 2).mean())), "tree_l2": float(np.sqrt((e_tree ** 2).mean())),
           "paper_direct_4threads_s": PAPER_DIRECT_4THREADS_S[ih]}
    rows.append(row)
    print(row, flush=True)
for a, b in zip(rows, rows[1:]):
    b["direct_slope"] = math.log(b["direct_ms"] / a["direct_ms"]) / math.log(b["N"] / a["N"])
    b["tree_slope"] = math.log(b["tree_ms"] / a["tree_ms"]) / math.log(b["N"] / a["N"])
out = {"what": "PAPER.md Fig. 6 on one B200 (spheroid SL, direct vs treecode with the eq. (33) policy)",
       "rows": rows}
if len(sys.argv) > 1:
    json.dump(out, open(sys.argv[1], "w"), indent=1)
print(json.dumps(rows[1:], indent=0))

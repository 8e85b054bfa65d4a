#!/usr/bin/env python
"""PAPER.md Table 2 (lines 357-365) on the GPU: two-drop IE (35) solves through
the C ABI at 1/h = 16 ... 128, GMRES iterations, self-convergence errors
e_h = u_h - u_{h/2} at the coarse nodes (eq. (36)) and their orders, and the
device time of each solve.  Writes the JSON to argv[1] (default stdout).

    python tools/twodrop_table2.py profiles/r01/twodrop_table2.json [levels...]
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2507_00156_b200 as ser  # noqa: E402
from workloads.twodrop import match_nodes, split, twodrop  # noqa: E402

args = [a for a in sys.argv[1:] if not a.startswith("--")]
use_tree = "--tree" in sys.argv  # every block through the treecode with Table 2's parameters
gap = next((float(a.split("=")[1]) for a in sys.argv if a.startswith("--xgap=")), None)  # (2+gap, 0, 0) drops
literal = "--literal" in sys.argv  # PAPER.md:339 as printed: centres (0,0,0), (2,0,1/16^3)
out_path = args[0] if args else None
levels = [int(a) for a in args[1:]] or [16, 32, 64, 128]


TABLE2 = {16: (1000, 6), 32: (1000, 6), 64: (2000, 8), 128: (4000, 10), 256: (8000, 12)}


def policy(inv_h):
    """Treecode parameters of PAPER.md Table 2 (theta 0.6, N0 and p per row, lines 359-363);
    other h: eq. (33) (h = 1/64: N0 2000, p 6; h -> h/2: N0 x 2, p + 2)."""
    if inv_h in TABLE2:
        return (*TABLE2[inv_h], 0.6)
    k = int(round(np.log2(inv_h / 64)))
    return (int(2000 * 2.0 ** k), max(2, 6 + 2 * k), 0.6)

rows, sol = [], {}
for ih in levels:
    if literal:
        td = twodrop(ih, separation="z")
    else:
        td = twodrop(ih) if gap is None else twodrop(ih, eps=gap, separation="x")
    t0 = time.perf_counter()
    s = ser.twodrop_solver(td, tree=policy(ih) if use_tree else None)
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    s.solve()  # warm-up (also checks convergence)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    u, it, hist = s.solve()
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    N = [d.N for d in td.drops]
    pairs_matvec = sum(N[i] * N[j] for i in range(2) for j in range(2))  # 4 blocks
    sol[ih] = (td, u.cpu().numpy())
    rows.append({"inv_h": ih, "N_per_drop": N, "tree": policy(ih) if use_tree else None, "iterations": it, "final_residual": hist[-1],
                 "solve_ms": ms, "setup_s": t_setup, "block_evals": 4 * (it + 1),
                 "pairs_per_solve": pairs_matvec * (it + 1),
                 "pairs_per_s": pairs_matvec * (it + 1) / (ms / 1e3), "u_max": float(np.abs(u.cpu().numpy()).max())})
    print(rows[-1], flush=True)
for r, r2 in zip(rows, rows[1:]):
    tc, uc = sol[r["inv_h"]]  # noqa
    tf, uf = sol[r2["inv_h"]]
    idx = match_nodes(tc, tf)
    c, f = split(tc, uc), split(tf, uf)
    e = np.concatenate([c[k] - f[k][:, idx[k]] for k in range(2)], axis=1)
    mag = np.linalg.norm(e, axis=0)
    r["max_err"] = float(mag.max())
    r["l2_err"] = float(np.sqrt((mag ** 2).sum() / e.shape[1]))
    xs = np.concatenate([d.x for d in tc.drops], axis=1)
    r["max_err_at"] = [float(v) for v in xs[:, int(np.argmax(mag))]]
    contact = 0.5 * (tc.drops[0].center + tc.drops[1].center)
    for rad in (0.1, 0.25, 0.5):
        away = np.linalg.norm(xs - contact[:, None], axis=0) > rad
        r[f"max_err_away_{rad}"] = float(mag[away].max())
for r, r2 in zip(rows, rows[1:]):
    if "max_err" in r and "max_err" in r2:
        r2["order_max"] = float(np.log2(r["max_err"] / r2["max_err"]))
        r2["order_l2"] = float(np.log2(r["l2_err"] / r2["l2_err"]))
        for rad in (0.1, 0.25, 0.5):
            k = f"max_err_away_{rad}"
            r2[f"order_away_{rad}"] = float(np.log2(r[k] / r2[k]))
c2 = [float(v) for v in sol[levels[0]][0].drops[1].center]
res = {"geometry": f"centres (0,0,0), {tuple(c2)}" + (" (PAPER.md:339 as printed)" if literal else
                                                     " (separation 2 + eps along x_1, DESIGN.md R17)"),
       "what": "PAPER.md Table 2 on one B200: two-drop IE (35), GMRES tol 1e-10, "
               + ("treecode (Table 2 parameters) on every block" if use_tree else "direct (no treecode) sums"),
       "paper_table2": {"16": [13, 3.17e-3, 1.19e-4], "32": [12, 1.07e-4, 6.11e-6], "64": [12, 4.06e-6, 2.11e-7],
                        "128": [12, 1.02e-7, 6.37e-9], "columns": ["iterations", "max err", "L2 err"]},
       "gpu": torch.cuda.get_device_name(), "rows": rows}
txt = json.dumps(res, indent=1)
if out_path:
    open(out_path, "w").write(txt)
print(txt)

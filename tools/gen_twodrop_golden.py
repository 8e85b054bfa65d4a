#!/usr/bin/env python
"""Write tests/golden/twodrop_oracle.json: the CPU oracle's two-drop solves
(Sec. 4.3, IE (35), GMRES tol 1e-10) at 1/h = 8, 16, 32 and the
self-convergence errors e_h = u_h - u_{h/2} at the coarse nodes (eq. (36)),
max and L2 (L2 = sqrt(sum |e|^2 / N), N = coarse node count; eq. (35)
`error_L2` reading).  Calls only oracle/ and workloads/.

    python tools/gen_twodrop_golden.py [--cache DIR]   (~10 min on 8 cores)
"""
import argparse
import json
import os
import pickle
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.twodrop import TwoDropOracle  # noqa: E402
from workloads.twodrop import match_nodes, split, twodrop  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--cache", default=None, help="reuse/store per-h solves as td_oracle_<inv_h>.pkl")
args = ap.parse_args()

levels = (8, 16, 32)
sol, its, hists, secs = {}, {}, {}, {}
for ih in levels:
    pk = os.path.join(args.cache, f"td_oracle_{ih}.pkl") if args.cache else None
    if pk and os.path.exists(pk):
        _, u, it, hist = pickle.load(open(pk, "rb"))
        dt = None
    else:
        t0 = time.time()
        u, it, hist = TwoDropOracle(twodrop(ih)).solve()
        dt = time.time() - t0
        if pk:
            pickle.dump((ih, u, it, hist), open(pk, "wb"))
    sol[ih], its[ih], hists[ih], secs[ih] = u, it, hist, dt
    print(ih, it, hist[-1], dt, flush=True)

max_err, l2_err = {}, {}
for a, b in zip(levels, levels[1:]):
    tc, tf = twodrop(a), twodrop(b)
    idx = match_nodes(tc, tf)
    uc, uf = split(tc, sol[a]), split(tf, sol[b])
    e = np.concatenate([(uc[k] - uf[k][:, idx[k]]) for k in range(2)], axis=1)  # (3, N_coarse)
    mag = np.linalg.norm(e, axis=0)
    max_err[a] = float(mag.max())
    l2_err[a] = float(np.sqrt((mag ** 2).sum() / e.shape[1]))
out = {"source": "oracle/twodrop.py (CPU, localized mode), tools/gen_twodrop_golden.py",
       "paper": "PAPER.md:357-365 Table 2 (treecode, other machine): max err 3.17e-3 (1/16), 1.07e-4 (1/32); "
                "L2 1.19e-4, 6.11e-6; iterations 13, 12, 12, 12",
       "norms": "max over coarse nodes of |e| (Euclidean 3-vector); L2 = sqrt(mean |e|^2)",
       "iterations": {str(k): v for k, v in its.items()},
       "final_residual": {str(k): v[-1] for k, v in hists.items()},
       "max_err": {str(k): v for k, v in max_err.items()},
       "l2_err": {str(k): v for k, v in l2_err.items()},
       "u_max": {str(k): float(np.abs(v).max()) for k, v in sol.items()}}
json.dump(out, open(os.path.join(ROOT, "tests", "golden", "twodrop_oracle.json"), "w"), indent=1)
print(json.dumps(out, indent=1))

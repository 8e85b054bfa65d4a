#!/usr/bin/env python
"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel.

    python tools/launch_summary.py gpurun_out/launches.csv [> profiles/rNN/launches_xxx.txt]
"""
import csv
import sys
from collections import defaultdict

lines = open(sys.argv[1]).read().splitlines()
start = [n for n, l in enumerate(lines) if l.startswith('"ID"')][0]
rows = list(csv.reader(lines[start:]))
h = rows[0]
iK, iV = h.index("Kernel Name"), h.index("Metric Value")
agg = defaultdict(lambda: [0, 0.0])
for r in rows[1:]:
    if len(r) != len(h):
        continue
    k = r[iK].split("(")[0][:80]
    agg[k][0] += 1
    agg[k][1] += float(r[iV].replace(",", ""))
tot = sum(v[1] for v in agg.values())
print(f"# {sys.argv[1]}: per-kernel totals (ncu, cold-cache serialised launches)")
print("launches      total_ms  share  kernel")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{v[0]:8d} {v[1] / 1e6:12.3f} {100 * v[1] / tot:5.1f}%  {k}")

#!/usr/bin/env python
"""Summarise an ncu report (.ncu-rep) into profiles/: key metrics per kernel as JSON.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep profiles/r02/ncu_full_xxx.json [bench_line.json]

With a bench line (the JSON bench.py printed for the SAME arguments without ncu), the
summary records that run's configuration as "bench_config"; bench.py takes
roofline.traffic only from a summary whose bench_config equals its own run.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum", "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum", "smsp__inst_executed.sum",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread", "launch__grid_size",
    "launch__block_size", "launch__shared_mem_per_block_static", "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
    "lts__t_sector_hit_rate.pct", "smsp__issue_active.avg.pct_of_peak_sustained_active",
]
STALL_PREFIX = "smsp__average_warps_issue_stalled_"


def bench_config(path):
    for line in open(path):
        if line.startswith("{"):
            c = json.loads(line)["config"]
            return {k: c.get(k) for k in ("workload", "path", "schedule", "targets_per_thread")}
    return None


def main(rep, out, bench_line=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = []
    for row in rows[2:]:
        k = {"kernel": row[hdr.index("Kernel Name")]}
        for i, name in enumerate(hdr):
            if name in KEYS:
                k[name] = f"{row[i]} {units[i]}".strip()
            elif name.startswith(STALL_PREFIX) and name.endswith("_per_issue_active.ratio"):
                v = row[i]
                try:
                    if float(v) > 0.01:
                        k.setdefault("stalls_per_issue", {})[name[len(STALL_PREFIX):-len("_per_issue_active.ratio")]] = float(v)
                except ValueError:
                    pass
        # FP64 op totals: this ncu reports the .sum of the SASS op counters only per elapsed cycle
        try:
            cyc = float(row[hdr.index("smsp__cycles_elapsed.avg")])
            for op in ("dfma", "dmul", "dadd"):
                name = f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum.per_cycle_elapsed"
                if name in hdr and f"smsp__sass_thread_inst_executed_op_{op}_pred_on.sum" not in k:
                    k[f"fp64_{op}_thread_inst_total"] = float(row[hdr.index(name)]) * cyc
        except (ValueError, IndexError):
            pass
        res.append(k)
    doc = {"report": rep, "kernels": res}
    if bench_line:
        doc["bench_config"] = bench_config(bench_line)
        doc["bench_line"] = bench_line
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=1)
    print(json.dumps(res, indent=1)[:3000])


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)

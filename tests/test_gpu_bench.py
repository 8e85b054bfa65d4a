"""bench.py's GPU arm keeps the driver's JSON-line contract (a short run on the B200):
every key the task names, the roofline and clock objects, and a positive launch count."""
from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--config", "5", "--inv-h", "64", "--steps", "3", "--warmup", "3",
                        "--no-cpu-baseline"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(s) for s in r.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "clocks", "gpu_launches", "e2e"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["value"] > 0
    assert d["dtype"] == "f64" and d["unit"] == "pairs/s" and "workload" in d["config"]
    ro = d["roofline"]
    assert ro["bound"] == "alu" and ro["unit"] == "TFLOP/s" and 0 < ro["frac"] < 1
    assert abs(ro["frac"] - ro["achieved"] / ro["peak"]) < 1e-9
    assert d["gpu_launches"] > 0
    e2e = d["e2e"]
    assert e2e["value"] > 0 and e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert "sm_mhz" in d["clocks"] and "reasons" in d["clocks"] and d["clocks"]["samples"] >= 3
    par = d["parity"]  # sampled parity against the oracle's definition mode, and the solve alone
    assert par["u_max_rel"] <= 1e-12 and par["v_max_rel"] <= 1e-12 and par["solve_max_rel"] <= 1e-13
    assert d["config"]["workload"] == "cfg5_sphere_h1/64"


@pytest.mark.gpu
@pytest.mark.parametrize("args", [["--config", "4", "--inv-h", "16", "--eps", "0.05"],
                                  ["--workload", "onsurface", "--inv-h", "16"],
                                  ["--workload", "tree", "--config", "5", "--inv-h", "32", "--tree", "500,4,0.6"]])
def test_bench_other_workloads(args):
    """The secondary bench workloads run and print one line with a positive value and a roofline."""
    r = subprocess.run([sys.executable, "bench.py", *args, "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(s) for s in r.stdout.splitlines() if s.startswith("{")]
    assert len(lines) == 1 and lines[0]["value"] > 0 and 0 < lines[0]["roofline"]["frac"] < 1
    par = lines[0]["parity"]  # every line carries its sampled oracle parity
    assert par["targets_sampled"] > 0 and max(par["u_max_rel"], par["v_max_rel"]) <= par["tolerance"] == 1e-12

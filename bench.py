#!/usr/bin/env python
"""Benchmark of the B200 hot path (BASELINE.json metric).

One step = one full SL+DL evaluation (3-delta localized regularization with the
fused extrapolation, stokes_er_eval) of BASELINE.json configs[4] at 1/h = 256:
the unit sphere's N = 1,090,854 quadrature nodes as sources and every node a
target (M = N, b = 0), rho = (2,3,4), seeded cubic densities -- the largest
single-GPU configuration, at N >= 1e5 where north_star states its bar.  Inputs
are resident in HBM when the timed region starts; L2 is flushed (256 MiB write)
between timed steps.  Other configs: --config 1..6 --inv-h H (6 = pure far).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line (rank 0).  Multi-GPU (torchrun, NCCL): ONE seeded target
set is split across the ranks (sharding.evaluate_sharded: contiguous ranges of
the Morton-sorted targets, sources replicated, one all-gather of u, v inside
the timed region) -- strong scaling, value =
the block's pairs / max-over-ranks device time.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "target-source pair interactions/sec (SL+DL, 3-delta extrap) & FP64 % of peak"
UNIT = "pairs/s"
# Stated per-pair FLOP counts: algorithmic
# flops with rsqrt/erf/exp = 1; FMA = 2.
F_FAR_ALG = 57
F_FAR_SL, F_FAR_DL = 35, 33  # SL-only / DL-only far pairs
F_NEAR_ALG = 180
# NEXT-1 s# near pair (one delta): y-x 3, r^2 5, rsqrt 1, r 1, t 1, erf 1, exp 1, t^2 t^3 t^5 3,
# s#1..3 polynomials 18, A1 A3 A5 5, SL 24, DL (unsplit, as the far pair) 21
F_NEAR_SHARP_ALG = 84
F_FAR_ISSUED = 64   # ncu-countable FP64 flops (2*DFMA + DMUL + DADD) of far_pair<3> (41 instructions)
F_NEAR_ISSUED = 331  # ncu-counted FP64 flops per near pair of near_kernel<3> incl. its classification (profiles/r02/ncu_full_near_cfg2_h64.json: 132.3 DFMA, 41.1 DMUL, 25.5 DADD = 199 instructions; round 1: 343)
# node-target path (csrc/sym.cuh): one evaluation of a far pair's shared part serves both directed
# pairs.  Algorithmic flops per UNORDERED pair (rsqrt = 1, FMA = 2): d 3, r^2 5, rsqrt 1, 1/r^2 and
# 1/r^5 3, SL 2 x 24, DL: q_j - q_i 3, d.dq 5, dq/r^5 1 shared + 2 x (d.mw 5, x 1, v += d c 6) = 93,
# i.e. 46.5 per directed pair (57 when each direction is computed alone).
F_SYM_UNORDERED_ALG = 93
F_SYM_UNORDERED_ISSUED = 99  # sym_pair<3> (unit-vector form): 60 FP64 instructions = 39 DFMA + 15 DMUL + 6 DADD (2*39 + 15 + 6)
SMS = 148
FP64_LANES_PER_SM = 64  # measured: DFMA loop 58.7 FMA/clk/SM at the boost clock (tools/probes)


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", type=int, default=5, help="BASELINE.json config index (1-based); default configs[4] (the N >= 1e5 sweep the north_star bar is stated at; 6 = pure-far micro-config)")
    ap.add_argument("--inv-h", type=int, default=256)
    ap.add_argument("--eps", type=float, default=0.05, help="config 4: centre separation 2 + eps")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--targets-per-thread", type=int, default=0)
    ap.add_argument("--near-phases", type=int, default=0)
    ap.add_argument("--chunk-tiles", type=int, default=0, help="far item = chunk x 128 sources (0: automatic)")
    ap.add_argument("--workload", choices=["eval", "twodrop", "tree", "onsurface"], default="eval",
                    help="eval: one stokes_er_eval of BASELINE.json config --config (default); "
                         "onsurface: one stokes_er_eval_onsurface (NEXT-1, s#, delta = 3h) of config 5 "
                         "(every node a target) at 1/h = --inv-h; "
                         "twodrop: one GMRES solve of the NEXT-2 two-drop IE (35) at 1/h = --inv-h; "
                         "tree: one stokes_er_eval_tree (NEXT-3) of config --config at 1/h = --inv-h")
    ap.add_argument("--tree", type=str, default="",
                    help="treecode N0,p,theta (default: PAPER.md eq. (33) policy for --inv-h)")
    ap.add_argument("--path", choices=["auto", "general", "nodes"], default="auto",
                    help="nodes: stokes_er_eval_nodes (targets = the nodes, symmetric far kernel); general: "
                         "stokes_er_eval; auto: nodes when the workload's targets are its nodes (config 5) on 1 GPU")
    ap.add_argument("--graph", choices=["auto", "on", "off"], default="auto",
                    help="time CUDA-graph replays of the evaluation (captured once after the warm-up; the same "
                         "kernels, without the per-call host enqueue on the timeline); auto: on for 1 GPU")
    ap.add_argument("--schedule", choices=["fused", "separate"], default="fused",
                    help="fused: one persistent kernel, far items and near items from one interleaved "
                         "queue (default); separate: far kernel then near kernel")
    return ap.parse_args()


def make_workload(cfg: int, inv_h: int, rank: int):
    from workloads.configs import config1, config2, config3, config5, pure_far
    seed = cfg + 1000 * rank
    if cfg == 6:  # pure-far micro-config isolating the far-field pair sum
        return pure_far(inv_h=inv_h, seed=seed)
    if cfg == 1:
        return config1(seed=seed)
    if cfg == 2:
        return config2(inv_h=inv_h, seed=seed)
    if cfg == 3:
        return config3(inv_h=inv_h, seed=seed)
    if cfg == 5:
        return config5(inv_h=inv_h, seed=seed)
    raise SystemExit("bench configs: 1, 2, 3, 5, 6 = pure far (config 4 has its own path: 4 blocks per step)")


def near_pair_count(block) -> int:
    """Pairs with r <= 6 delta_max (the near rule of include/stokes_er.h), by KD-tree."""
    from scipy.spatial import cKDTree
    rc = 6.0 * max(block.rho) * block.h
    counts = cKDTree(block.src_xyz.T).query_ball_point(block.tgt_xyz.T, rc, return_length=True, workers=-1)
    return int(np.asarray(counts, dtype=np.int64).sum())


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 3.0:  # sampler running before the timed region
                time.sleep(0.01)
        except OSError:
            self.proc = None
        return self

    def pad(self, busy, min_samples=5, limit_s=5.0, agree=None):
        """Short timed regions see few 50 ms samples: keep the GPU busy with untimed steps
        (`busy()`) until the record holds `min_samples` (clocks under the same load).
        `agree(flag) -> bool` (multi-rank runs) makes every rank take the same decision, so
        ranks whose steps run collectives stay in step."""
        t0 = time.time()
        while True:
            need = self.proc is not None and len(self.lines) < min_samples and time.time() - t0 < limit_s
            if agree is not None:
                need = agree(need)
            if not need:
                return
            busy()

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self.t.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[4:8]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def run_reference(args, rank, world):
    """--impl reference: the CPU oracle (localized mode = the paper's algorithm) as it
    stands, on the host cores, rank 0 only; each step a bounded target sample."""
    if rank != 0:
        return None
    import oracle
    block = make_workload(args.config, args.inv_h, 0)
    cores = oracle.max_threads()
    rng = np.random.default_rng(0)
    k = 256
    t0 = time.perf_counter()
    oracle.evaluate_block(block.take_targets(rng.choice(block.M, k, replace=False)), localized=True)
    per_target = (time.perf_counter() - t0) / k
    k = int(min(block.M, max(64, 0.4 / per_target)))  # ~0.4 s per step
    times, pairs = [], 0
    for it in range(args.warmup + args.steps):
        idx = rng.choice(block.M, k, replace=False)
        sub = block.take_targets(idx)
        t0 = time.perf_counter()
        oracle.evaluate_block(sub, localized=True)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
            pairs += k * block.N
    total = sum(times)
    value = pairs / total
    cpu = {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{k} random targets of {block.M} per step x all {block.N} sources, localized mode "
                     f"(shared far field, PAPER.md:183-191), {args.steps} steps"}
    return {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic", "impl": "reference",
            "config": {"workload": block.name, "N": block.N, "M": block.M, "h": block.h, "rho": list(block.rho)},
            "cpu_baseline": cpu, "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                                         "d2h_bytes_per_step": 0}}


def twodrop_launches(it: int) -> int:
    """Our kernel launches in one stokes_er_twodrop_solve that took `it` Krylov steps."""
    per_blocks = 2 * (8 + 7)                # self block (node path, 8) + cross block (7) per drop
    n = per_blocks + 2 + 2 + 1              # rhs: 4 block evals + 2 combines, norm (2), scale (1)
    for j in range(it):
        n += per_blocks + 2 + 2             # operator: 4 evals, 2 interpolations, 2 combines
        n += 3 * (j + 1) + 3                # MGS: dot (2) + update (1) per basis vector; norm (2) + scale (1)
    return n + it                           # u = V y

F_PROXY_ALG = 77  # algorithmic flops of one target-proxy interaction of eq. (31): a far pair's 57 with the
                  # DL contraction over the 9 q_a n_c w channels (41 flops) in place of the 3-vector form (21)


def run_tree(args, rank, world):
    """NEXT-3 bench: one step = one stokes_er_eval_tree (plan reused: the octree depends on the
    nodes only) of config --config at 1/h = --inv-h; value = direct-equivalent pair
    interactions per second (M N / time); accuracy against the direct path in the same run."""
    import ctypes

    import torch

    import paper_2507_00156_b200 as ser

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    block = make_workload(args.config, args.inv_h, rank)
    M, N = block.M, block.N
    if args.tree:
        n0, p, th = args.tree.split(",")
        tp = (int(n0), int(p), float(th))
    else:  # PAPER.md eq. (33): theta 0.6, N0 2000 and p 6 at h = 1/64, N0 x 2 and p + 2 per halving
        k = int(round(math.log2(args.inv_h / 64)))
        tp = (int(2000 * 2.0 ** k), max(2, 6 + 2 * k), 0.6)
    t0 = time.perf_counter()
    plan = ser.TreePlan(block.src_xyz, *tp)
    t_plan = time.perf_counter() - t0
    arrs = ser.to_device(block, dev)
    u = torch.empty((3, M), dtype=torch.float64, device=dev)
    v = torch.empty((3, M), dtype=torch.float64, device=dev)
    nbytes = int(ser._lib.load().stokes_er_tree_workspace_bytes(M, N, 3, ctypes.byref(plan.params), plan.ptr()))
    ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    K, W = args.steps, args.warmup
    for _ in range(W):
        flush.zero_()
        ser.evaluate_tree(*arrs, block.h, block.rho, plan, out_u=u, out_v=v, workspace=ws)
    torch.cuda.synchronize(dev)
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(K):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            ser.evaluate_tree(*arrs, block.h, block.rho, plan, out_u=u, out_v=v, workspace=ws)
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
    from paper_2507_00156_b200.sharding import max_over_ranks
    total_s = max_over_ranks(sum(ms) / 1e3, dev)
    ud, vd = ser.evaluate(*arrs, block.h, block.rho)
    torch.cuda.synchronize(dev)
    diff = max(float((u - ud).abs().max() / ud.abs().max()), float((v - vd).abs().max() / vd.abs().max()))
    if rank != 0:
        return None
    # work counts from the treecode oracle on a target sample (per-target traversal statistics)
    import oracle
    rng = np.random.default_rng(0)
    idx = rng.choice(M, min(M, 128), replace=False)
    ut, vt, st = oracle.evaluate_tree_block(block.take_targets(idx), leaf_size=tp[0], degree=tp[1], theta=tp[2],
                                            stats=True)
    ug, vg = u.cpu().numpy()[:, idx], v.cpu().numpy()[:, idx]
    parity = {"u_max_rel": float(np.abs(ug - ut).max() / np.abs(ut).max()),
              "v_max_rel": float(np.abs(vg - vt).max() / np.abs(vt).max()), "targets_sampled": int(len(idx)),
              "sample_seed": 0, "reference": "oracle treecode (oracle_eval_tree, same N0, p, theta), same seeded inputs",
              "tolerance": 1e-12}
    proxies = st[1] / len(idx) * (tp[1] + 1) ** 3 * M
    direct = st[2] / len(idx) * M
    near = near_pair_count(block)
    flops = proxies * F_PROXY_ALG + (direct - near) * F_FAR_ALG + near * F_NEAR_ALG
    peak = SMS * FP64_LANES_PER_SM * 2 * 1965.0 * 1e6 / 1e12
    achieved = flops / (total_s / K) / 1e12
    line = {"metric": "treecode (NEXT-3) SL+DL 3-delta evaluation: direct-equivalent pair interactions/sec (M N / time)",
            "value": world * M * N * K / total_s, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * total_s / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": block.name + "_treecode", "N": N, "M": M, "N0": tp[0], "p": tp[1],
                       "theta": tp[2], "tree_nodes": plan.nodes, "tree_depth": plan.depth,
                       "host_plan_build_s": t_plan, "max_rel_diff_vs_direct": diff,
                       "proxy_interactions_per_step": proxies, "direct_pairs_per_step": direct,
                       "near_pairs_per_step": near, "work_counts": "oracle traversal statistics on 128 targets",
                       "l2": "flushed between timed steps (256 MiB write)", "inputs": "resident in HBM"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "whole treecode evaluation (P2M/M2M, tree walk + near units, finalize): "
                                   f"{F_PROXY_ALG} flops per target-proxy interaction, {F_FAR_ALG} per direct far "
                                   f"pair, {F_NEAR_ALG} per near pair",
                         "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk/SM x 2 x 1965 MHz"},
            "clocks": clk.summary(), "parity": parity, "gpu_launches": K * 9,
            "gpu_launches_note": "per step: bbox, morton, pack sources, pack targets, P2M, M2M per level (<= 3), "
                                 "tree walk + near units, finalize (+ CUB sort)",
            "e2e": None}
    return line


def run_onsurface(args, rank, world):
    """NEXT-1 bench: one step = one stokes_er_eval_onsurface (s# factors, one delta = 3h, cutoff 7;
    PAPER.md:126-139 and 341) of config 5 (M = N: every sphere node is a target, b = 0) at
    1/h = --inv-h; value = pair interactions per second (M N / time)."""
    import torch
    from scipy.spatial import cKDTree

    import paper_2507_00156_b200 as ser

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    block = make_workload(5, args.inv_h, rank)
    M, N = block.M, block.N
    delta = 3.0 * block.h
    arrs = ser.to_device(block, dev)
    u = torch.empty((3, M), dtype=torch.float64, device=dev)
    v = torch.empty((3, M), dtype=torch.float64, device=dev)
    # every node is a target: the node path (symmetric far kernel) from 5e4 nodes on, as the two-drop
    # self blocks; stokes_er_eval_onsurface below
    nodes = args.path == "nodes" or (args.path == "auto" and N >= 50000)
    if nodes:
        ws = torch.empty(ser.nodes_workspace_bytes(N, 3), dtype=torch.uint8, device=dev)
        run = lambda: ser.evaluate_nodes_onsurface(*arrs[:5], delta, out_u=u, out_v=v, workspace=ws)
    else:
        ws = ser.alloc_workspace(M, N, 3, dev)
        run = lambda: ser.evaluate_onsurface(*arrs, delta, out_u=u, out_v=v, workspace=ws)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    K, W = args.steps, args.warmup
    for _ in range(W):
        flush.zero_()
        run()
    torch.cuda.synchronize(dev)
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(K):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            run()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
    from paper_2507_00156_b200.sharding import max_over_ranks
    total_s = max_over_ranks(sum(ms) / 1e3, dev)
    if rank != 0:
        return None
    near = int(cKDTree(block.tgt_xyz.T).count_neighbors(cKDTree(block.src_xyz.T), 7.0 * delta))
    flops = (M * N - near) * F_FAR_ALG + near * F_NEAR_SHARP_ALG
    peak = SMS * FP64_LANES_PER_SM * 2 * 1965.0 * 1e6 / 1e12
    achieved = flops / (total_s / K) / 1e12
    line = {"metric": "on-surface s# (NEXT-1) SL+DL evaluation: target-source pair interactions/sec",
            "value": world * M * N * K / total_s, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * total_s / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": block.name + "_onsurface", "N": N, "M": M, "delta_over_h": 3.0, "cutoff": 7.0,
                       "path": "stokes_er_eval_nodes_onsurface" if nodes else "stokes_er_eval_onsurface",
                       "near_pairs_per_step": near, "l2": "flushed between timed steps (256 MiB write)",
                       "inputs": "resident in HBM"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": f"the whole evaluation: {F_FAR_ALG} flops per far pair, {F_NEAR_SHARP_ALG} per "
                                   "s# near pair (rsqrt, erf, exp = 1)" + (" -- counted per directed far pair; the "
                                   "node path evaluates each pair's geometry once for both directions (46.5 "
                                   "honest flops per directed pair, DESIGN.md 5.7)" if nodes else ""),
                         "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk/SM x 2 x 1965 MHz"},
            "clocks": clk.summary(), "gpu_launches": K * (ser.nodes_launch_count(N) if nodes else ser.launch_count(M, N)),
            "gpu_launches_note": ("per step: bbox, morton, pack_sources, pack_node_soa, block_boxes, sym_kernel, "
                                  "nbr_kernel, finalize_nodes (+ CUB sort)" if nodes else
                                  "per step: bbox, 2 morton, pack sources, pack targets, fused far+near, finalize "
                                  "(+ CUB sort)"),
            "e2e": None}
    # the oracle's sharp mode on a target sample, host cores: the CPU baseline (a ~2e9-pair sample) and the
    # sampled parity (16 targets when the baseline is off)
    import oracle
    rng = np.random.default_rng(0)
    k = 16 if args.no_cpu_baseline else max(64, min(M, int(2e9 / N)))
    idx = np.sort(rng.choice(M, min(M, k), replace=False))
    sub = block.take_targets(idx)
    t0 = time.perf_counter()
    ur, vr = oracle.evaluate_sharp(*sub.arrays(), delta, localized=True, cutoff=7.0)
    dt = time.perf_counter() - t0
    uu, vv = u.cpu().numpy()[:, idx], v.cpu().numpy()[:, idx]
    line["parity"] = {"u_max_rel": float(np.abs(uu - ur).max() / np.abs(ur).max()),
                      "v_max_rel": float(np.abs(vv - vr).max() / np.abs(vr).max()),
                      "targets_sampled": int(len(idx)), "sample_seed": 0,
                      "reference": "oracle s# mode (oracle_eval_sharp, cutoff 7), same seeded inputs",
                      "tolerance": 1e-12}
    line["config"]["max_rel_diff_vs_oracle_sample"] = max(line["parity"]["u_max_rel"], line["parity"]["v_max_rel"])
    if not args.no_cpu_baseline:
        line["cpu_baseline"] = {"value": len(idx) * N / dt, "unit": UNIT, "cores": oracle.max_threads(),
                                "kind": "oracle",
                                "sample": f"{len(idx)} random targets of {M} x all {N} sources, sharp mode, "
                                          f"localized, {dt:.1f} s wall"}
    return line


def run_config4(args, rank, world):
    """BASELINE.json config 4: two unit spheres at centre separation 2 + eps (--eps), 1/h = --inv-h;
    one step = the 4 block evaluations of the two-sphere field (A<-A, A<-B, B<-A, B<-B, each a
    stokes_er_eval with targets = the nodes of one sphere); value = sum of the blocks' M N per second."""
    import torch
    from scipy.spatial import cKDTree

    import paper_2507_00156_b200 as ser
    from workloads.configs import config4

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    blocks = config4(eps=args.eps, inv_h=args.inv_h, seed=4 + 1000 * rank)
    dblocks = [ser.to_device(b, dev) for b in blocks]
    outs = [(torch.empty((3, b.M), dtype=torch.float64, device=dev), torch.empty((3, b.M), dtype=torch.float64,
                                                                                  device=dev)) for b in blocks]
    wss = [ser.alloc_workspace(b.M, b.N, 3, dev) for b in blocks]
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)

    def step():
        for b, arrs, (u, v), ws in zip(blocks, dblocks, outs, wss):
            ser.evaluate(*arrs, b.h, b.rho, out_u=u, out_v=v, workspace=ws)

    K, W = args.steps, args.warmup
    for _ in range(W):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(K):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            step()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
    from paper_2507_00156_b200.sharding import max_over_ranks
    total_s = max_over_ranks(sum(ms) / 1e3, dev)
    if rank != 0:
        return None
    pairs = sum(b.M * b.N for b in blocks)
    near = sum(int(cKDTree(b.tgt_xyz.T).count_neighbors(cKDTree(b.src_xyz.T), 6.0 * max(b.rho) * b.h))
               for b in blocks)
    flops = (pairs - near) * F_FAR_ALG + near * F_NEAR_ALG
    peak = SMS * FP64_LANES_PER_SM * 2 * 1965.0 * 1e6 / 1e12
    achieved = flops / (total_s / K) / 1e12
    line = {"metric": METRIC, "value": world * pairs * K / total_s, "unit": UNIT, "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": 1e3 * total_s / K, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"cfg4_two_spheres_eps{args.eps}_h1/{args.inv_h}", "N_per_sphere": blocks[0].N,
                       "blocks": [b.name for b in blocks], "pairs_per_step": pairs, "near_pairs_per_step": near,
                       "rho": list(blocks[0].rho), "l2": "flushed between timed steps (256 MiB write)",
                       "inputs": "resident in HBM"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": f"the 4 evaluations: {F_FAR_ALG} flops per far pair, {F_NEAR_ALG} per near pair",
                         "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk/SM x 2 x 1965 MHz"},
            "clocks": clk.summary(), "gpu_launches": K * 4 * 7,
            "gpu_launches_note": "per block: bbox, 2 morton, pack sources, pack targets, fused far+near, finalize "
                                 "(+ CUB sort)",
            "e2e": None}
    # sampled parity of each block's output (after the timed region) against the oracle's definition mode
    recs = [sampled_parity(b, u.cpu().numpy(), v.cpu().numpy(), n=16)[0] for b, (u, v) in zip(blocks, outs)]
    line["parity"] = {"u_max_rel": max(r["u_max_rel"] for r in recs), "v_max_rel": max(r["v_max_rel"] for r in recs),
                      "targets_sampled": sum(r["targets_sampled"] for r in recs), "sample_seed": recs[0]["sample_seed"],
                      "reference": recs[0]["reference"] + " (16 targets per block, max over the 4 blocks)",
                      "tolerance": recs[0]["tolerance"]}
    if not args.no_cpu_baseline:
        import oracle
        rng = np.random.default_rng(0)
        t_cpu, p_cpu = 0.0, 0
        for b in blocks:  # ~2.5 s of oracle work per block
            k = max(32, min(b.M, int(5e8 / b.N)))
            sub = b.take_targets(np.sort(rng.choice(b.M, k, replace=False)))
            t0 = time.perf_counter()
            oracle.evaluate_block(sub, localized=True)
            t_cpu += time.perf_counter() - t0
            p_cpu += k * b.N
        line["cpu_baseline"] = {"value": p_cpu / t_cpu, "unit": UNIT, "cores": oracle.max_threads(), "kind": "oracle",
                                "sample": f"random target samples of each of the 4 blocks, localized mode, "
                                          f"{t_cpu:.1f} s wall"}
    return line


def run_twodrop(args, rank, world):
    """NEXT-2 bench: one step = one full GMRES solve of IE (35) (Sec. 4.3)
    on the two drops at 1/h = args.inv_h through stokes_er_twodrop_solve: 4 block
    evaluations per Krylov step + the right-hand side, tol 1e-10.  value = block
    pair interactions per second (4 blocks x (iterations + 1) x N_b N_m pairs / time)."""
    import torch

    import paper_2507_00156_b200 as ser
    from workloads.twodrop import twodrop

    dist = None
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)
    td = twodrop(args.inv_h)
    N = [d.N for d in td.drops]
    s = ser.twodrop_solver(td, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    K, W = args.steps, args.warmup
    iters = []
    for _ in range(W):
        flush.zero_()
        s.solve()
    torch.cuda.synchronize(dev)
    if dist is not None:
        dist.barrier()
    ms = []
    with ClockSampler(local) as clk:
        for _ in range(K):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record()
            _, it, hist = s.solve()
            b.record()
            b.synchronize()
            ms.append(a.elapsed_time(b))
            iters.append(it)
    from paper_2507_00156_b200.sharding import max_over_ranks
    total_s = max_over_ranks(sum(ms) / 1e3, dev)
    pairs_matvec = sum(N[i] * N[j] for i in range(2) for j in range(2))
    it = iters[-1]
    pairs = pairs_matvec * (it + 1)
    value = world * pairs * K / total_s
    # end to end through the public API: host arrays -> device, setup, solve, u -> host
    e_ms = []
    host = [np.ascontiguousarray(a) for d in td.drops for a in (d.x, d.n, d.w, d.f)]
    h2d = sum(a.nbytes for a in host) + sum(c.b.nbytes + c.n0.nbytes + c.f0.nbytes for c in td.cross)
    for _ in range(max(3, K // 4)):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        s2 = ser.twodrop_solver(td, device=dev)
        u, _, _ = s2.solve()
        u_host = u.cpu()
        b.record()
        b.synchronize()
        e_ms.append(a.elapsed_time(b))
    e_total = max_over_ranks(sum(e_ms) / 1e3, dev)
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None
    # algorithmic flops of the solve's block evaluations (near pairs by KD-tree per block)
    from scipy.spatial import cKDTree
    near = 0
    for b in range(2):
        tb = cKDTree(td.drops[b].x.T)
        near += tb.count_neighbors(cKDTree(td.drops[b].x.T), 7.0 * td.delta_self)        # self: s#, c = 7
        near += tb.count_neighbors(cKDTree(td.drops[1 - b].x.T), 6.0 * max(td.rho) * td.h)  # cross: c = 6
    near *= (it + 1)
    # the rhs evaluates SL-only blocks, every Krylov step DL-only blocks: count every
    # pair (near ones included, a lower bound) at the far-pair flops of its mode
    flops = pairs_matvec * (F_FAR_SL + F_FAR_DL * it)
    peak = SMS * FP64_LANES_PER_SM * 2 * 1965.0 * 1e6 / 1e12
    achieved = flops / (total_s / K) / 1e12
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        from oracle.twodrop import TwoDropOracle
        tds = twodrop(min(args.inv_h, 16))
        o = TwoDropOracle(tds)
        vec = np.random.default_rng(0).uniform(-1, 1, tds.n_unknowns)
        t0 = time.perf_counter()
        o.apply(vec)
        dt = time.perf_counter() - t0
        Ns = [d.N for d in tds.drops]
        # parity of the operator (the solve's only kernel path) on the same small instance and vector
        got = ser.twodrop_solver(tds, device=dev).apply(torch.from_numpy(vec).to(dev)).cpu().numpy()
        ref = o.apply(vec)
        parity = {"apply_max_rel": float(np.abs(got - ref).max() / np.abs(ref).max()),
                  "instance": f"1/h = {min(args.inv_h, 16)}, seeded vector U[-1,1]",
                  "reference": "oracle/twodrop.py operator application (localized mode)", "tolerance": 1e-12}
        cpu = {"value": sum(Ns[i] * Ns[j] for i in range(2) for j in range(2)) / dt, "unit": UNIT,
               "cores": __import__("oracle").max_threads(), "kind": "oracle",
               "sample": f"one operator application (4 blocks) of the oracle at 1/h = {min(args.inv_h, 16)} "
                         f"(N = {Ns[0]} per drop), localized mode, {dt:.1f} s wall"}
    line = {"metric": "two-drop IE (35) GMRES solve: block pair interactions/sec (SL+DL blocks, tol 1e-10)",
            "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * total_s / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": f"twodrop_h1/{args.inv_h}", "N_per_drop": N, "iterations": it,
                       "block_evals_per_solve": 4 * (it + 1), "pairs_per_solve": pairs,
                       "near_pairs_per_solve": int(near), "rho_cross": list(td.rho), "delta_self_over_h": 3.0,
                       "eps": td.meta["eps"], "centre_2": [float(c) for c in td.drops[1].center], "lambda": list(td.meta["lambda"]), "tol": td.tol,
                       "l2": "flushed between timed steps (256 MiB write)", "inputs": "resident in HBM",
                       "parallelism": f"replicas x{world}"},
            "roofline": {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
                         "frac": achieved / peak, "traffic": None,
                         "kernel": "whole solve (4 (it+1) stokes_er_eval calls + GMRES vector ops) over its "
                                   "device time: every pair at the far-pair algorithmic flops of its mode, "
                                   f"{F_FAR_SL} (SL, rhs) / {F_FAR_DL} (DL, Krylov steps); a lower bound",
                         "peak_source": "derived: 148 SMs x 64 FP64 FMA/clk/SM x 2 x 1965 MHz"},
            "clocks": clk.summary(),
            "gpu_launches": K * twodrop_launches(it),
            "gpu_launches_note": "per solve: rhs (4 evals x 7 + 2 combines) + per Krylov step j (4 evals x 7 + "
                                 "2 interpolations + 2 combines + (j+1) MGS dots/updates x 3 + norm/scale 3) + "
                                 "final combination (our kernels; CUB sort launches not counted)",
            "e2e": {"value": world * pairs * len(e_ms) / e_total, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(u_host.numel() * 8),
                    "note": "host arrays -> device, stencil setup, solve, u -> host"}}
    if cpu:
        line["cpu_baseline"] = cpu
        line["parity"] = parity
    if dist is not None:
        dist.destroy_process_group()
    return line


def committed_traffic(bench_cfg: dict, kernel_prefix: str):
    """DRAM bytes (read + write) per launch of the dominant kernel from a committed
    `ncu --set full` summary (profiles/*/ncu_full_*.json) whose recorded bench
    configuration equals this run's (workload, path, schedule, targets per thread);
    None when no capture of this exact command exists."""
    import glob
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    keys = ("workload", "path", "schedule", "targets_per_thread")
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "ncu_full_*.json")), reverse=True):
        try:
            d = json.load(open(path))
        except (OSError, ValueError):
            continue
        meta = d.get("bench_config")
        if not meta or any(meta.get(k) != bench_cfg.get(k) for k in keys):
            continue
        want = kernel_prefix.replace("ser::", "")  # ncu's raw page prints the name without the namespace
        for k in d.get("kernels", []):
            if k["kernel"].replace("ser::", "").startswith(want) and "dram__bytes_read.sum" in k:
                tot = 0.0
                for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                    v, u = k[key].split()
                    tot += float(v.replace(",", "")) * units[u]
                return int(tot), os.path.relpath(path, ROOT) + " (ncu capture of this bench configuration)"
    return None


def sampled_parity(block, u_gpu, v_gpu, n=48, seed=7):
    """Max-norm relative error of the GPU output against the oracle's DEFINITION mode
    (every pair regularized for every delta: the parity reference) on a seeded sample
    of n targets x all N sources.  Returns (record, oracle seconds, pairs)."""
    import oracle
    rng = np.random.default_rng(seed)
    idx = np.sort(rng.choice(block.M, min(n, block.M), replace=False))
    sub = block.take_targets(idx)
    t0 = time.perf_counter()
    ur, vr = oracle.evaluate_block(sub, localized=False)
    dt = time.perf_counter() - t0
    eu = float(np.abs(u_gpu[:, idx] - ur).max() / np.abs(ur).max())
    ev = float(np.abs(v_gpu[:, idx] - vr).max() / np.abs(vr).max())
    return {"u_max_rel": eu, "v_max_rel": ev, "targets_sampled": int(len(idx)), "sample_seed": seed,
            "reference": "oracle definition mode (every pair, every delta), same seeded inputs",
            "tolerance": 1e-12}, dt, len(idx) * block.N


def solve_parity(block, dev, stream):
    """The 3x3 extrapolation solve alone (stokes_er_extrapolate vs the oracle's pivoted
    elimination) on seeded per-delta values: the workload's own b values (a sample) and
    b spread over [-6 delta_3, 6 delta_3]; tolerance 1e-13 (north_star)."""
    import torch

    import oracle
    import paper_2507_00156_b200 as ser
    rng = np.random.default_rng(11)
    b = np.concatenate([rng.choice(block.tgt_b, 128),
                        rng.uniform(-6, 6, 128) * max(block.rho) * block.h, [0.0]])
    ind = rng.uniform(-1, 1, (3, 6, b.size))
    got = ser.extrapolate(torch.from_numpy(b).to(dev), block.h, block.rho, torch.from_numpy(ind).to(dev),
                          stream=stream).cpu().numpy()
    ref = oracle.extrapolate(b, block.h, block.rho, ind)
    return float(np.abs(got - ref).max() / np.abs(ref).max())


def cpu_baseline(block, definition=None):
    """The oracle on the host cores, as it stands, on bounded target samples:
    localized mode (the paper's shared-far-field algorithm) on all cores is
    `value`; definition mode (every pair regularized: the parity reference) and one-core
    timings of both modes sit beside it.  ~20 s of CPU work in total."""
    import oracle
    cores = oracle.max_threads()
    rng = np.random.default_rng(1)

    def rate(localized, nthreads, budget_s):
        k, dt = 4, 0.0
        while dt < 0.1 * budget_s and k < block.M:  # calibrate on a growing sample (thread start-up amortised)
            k = min(block.M, 2 * k)
            t0 = time.perf_counter()
            oracle.evaluate_block(block.take_targets(rng.choice(block.M, k, replace=False)), localized=localized,
                                  nthreads=nthreads)
            dt = time.perf_counter() - t0
        k = int(min(block.M, max(8, budget_s * k / max(dt, 1e-9))))
        idx = rng.choice(block.M, k, replace=False)
        t0 = time.perf_counter()
        oracle.evaluate_block(block.take_targets(idx), localized=localized, nthreads=nthreads)
        dt = time.perf_counter() - t0
        return k * block.N / dt, k, dt

    v, k, dt = rate(True, 0, 10.0)
    rec = {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle",
           "sample": f"{k} random targets of {block.M} x all {block.N} sources, localized mode "
                     f"(the paper's shared-far-field algorithm, P:183-191), {dt:.1f} s wall on {cores} threads"}
    if definition is not None:
        dsec, dpairs = definition
        rec["definition_mode"] = {"value": dpairs / dsec, "unit": UNIT, "cores": cores,
                                  "sample": f"the parity sample ({dpairs // block.N} targets x all sources), "
                                            f"{dsec:.1f} s wall"}
    v1, k1, dt1 = rate(True, 1, 4.0)
    rec["one_core_localized"] = {"value": v1, "unit": UNIT, "cores": 1,
                                 "sample": f"{k1} targets x all sources, {dt1:.1f} s wall"}
    v2, k2, dt2 = rate(False, 1, 4.0)
    rec["one_core_definition"] = {"value": v2, "unit": UNIT, "cores": 1,
                                  "sample": f"{k2} targets x all sources, {dt2:.1f} s wall"}
    try:
        model = [l.split(":", 1)[1].strip() for l in open("/proc/cpuinfo") if l.startswith("model name")][0]
    except (OSError, IndexError):
        model = None
    rec["cpu_model"] = model
    return rec


def sharded_step(arrs, block, evaluate_fn):
    """The multi-rank step of run_eval: this rank's Morton range of ONE target set against
    all sources, then the all-gather of u, v back into the caller's order
    (sharding.evaluate_sharded)."""
    from paper_2507_00156_b200 import sharding
    return sharding.evaluate_sharded(*arrs, block.h, block.rho, mode=3, gather=True, evaluate_fn=evaluate_fn)


def nodes_sharded_step(src_arrs, block, opt, ws, stream):
    """The multi-rank node-path step: shard `rank` of the symmetric evaluation, then the all-reduce
    of u, v (sharding.evaluate_nodes_sharded)."""
    from paper_2507_00156_b200 import sharding
    return sharding.evaluate_nodes_sharded(*src_arrs, block.h, block.rho, mode=3, options=opt, workspace=ws,
                                           stream=stream)


def run_eval(args, rank, world):
    """The default bench: one step = one full SL+DL 3-delta evaluation of BASELINE.json
    config --config at 1/h = --inv-h (default config 5 at 1/h = 256: the unit sphere's
    N = M = 1,090,854 nodes, every node a target at b = 0).  Config 5's targets are its
    nodes, so on one GPU the step is stokes_er_eval_nodes (the same sums with the symmetric
    far kernel); other configs, or --path general, use stokes_er_eval.

    N = 1: one process evaluates the whole block.  N > 1 (torchrun, NCCL): ONE seeded
    target set split across the ranks by sharding.evaluate_sharded (contiguous ranges
    of the Morton-sorted targets, sources replicated, the all-gather of u, v inside the
    timed region) -- strong scaling, value = the
    block's M N pairs / max-over-ranks time."""
    import ctypes

    import torch

    import paper_2507_00156_b200 as ser
    from paper_2507_00156_b200.sharding import max_over_ranks, shard_bounds

    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device(f"cuda:{local}"))
    dev = torch.device(f"cuda:{local}")
    torch.cuda.set_device(dev)

    block = make_workload(args.config, args.inv_h, 0)  # one target set for every rank (strong scaling)
    M, N = block.M, block.N
    pairs = M * N
    a0, a1 = shard_bounds(M, rank, world)
    M_loc = a1 - a0
    arrs = ser.to_device(block, dev)
    opt = ser.Options()
    if args.targets_per_thread:
        opt.targets_per_thread = args.targets_per_thread
    if args.near_phases:
        opt.near_phases = args.near_phases
    if args.chunk_tiles:
        opt.source_chunk_tiles = args.chunk_tiles
    fused = args.schedule != "separate"
    opt.schedule = {"fused": 0, "separate": 1}[args.schedule]
    L = ser._lib.load()
    # auto: the node path for config 5 on one GPU from N ~ 1.5e5 on (below that the general path is faster:
    # 1/h = 64: 17.8 vs 15.9 ms; 1/h = 128: 204 vs 211 ms; 1/h = 256: 2.93 vs 3.25 s)
    nodes = args.path == "nodes" or (args.path == "auto" and args.config == 5 and N >= 150000)
    if nodes and args.config != 5:
        raise SystemExit("--path nodes: node-target workloads (config 5)")
    if nodes:
        ws = torch.empty(ser.nodes_workspace_bytes(N, 3, opt), dtype=torch.uint8, device=dev)
    else:
        ws = torch.empty(int(L.stokes_er_workspace_bytes_ex(M_loc, N, 3, ctypes.byref(opt))), dtype=torch.uint8,
                         device=dev)
    out_u = torch.empty((3, M), dtype=torch.float64, device=dev)
    out_v = torch.empty((3, M), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    K, W = args.steps, args.warmup

    def local_eval(sx, sn, sw, f, q, ty, tb, tx, h, rho, mode=3, ev_pair=None, ev_near=None, ou=None, ov=None):
        opt.pair_kernel_start_event = ev_pair[0].cuda_event if ev_pair else None
        opt.pair_kernel_end_event = ev_pair[1].cuda_event if ev_pair else None
        opt.near_kernel_start_event = ev_near[0].cuda_event if ev_near else None
        opt.near_kernel_end_event = ev_near[1].cuda_event if ev_near else None
        return ser.evaluate(sx, sn, sw, f, q, ty, tb, tx, h, rho, mode=mode, out_u=ou, out_v=ov, workspace=ws,
                            stream=torch.cuda.current_stream(dev), options=opt)

    def step(ev_pair=None, ev_near=None):
        if nodes:
            opt.pair_kernel_start_event = ev_pair[0].cuda_event if ev_pair else None
            opt.pair_kernel_end_event = ev_pair[1].cuda_event if ev_pair else None
            opt.near_kernel_start_event = ev_near[0].cuda_event if ev_near else None
            opt.near_kernel_end_event = ev_near[1].cuda_event if ev_near else None
            if world > 1:  # shard r of the block-pair items + one all-reduce of u, v
                return nodes_sharded_step(arrs[:5], block, opt, ws, stream)
            ser.evaluate_nodes(*arrs[:5], block.h, block.rho, out_u=out_u, out_v=out_v, workspace=ws,
                               stream=torch.cuda.current_stream(dev), options=opt)
            return out_u, out_v
        if world == 1:
            local_eval(*arrs, block.h, block.rho, ev_pair=ev_pair, ev_near=ev_near, ou=out_u, ov=out_v)
            return out_u, out_v
        return sharded_step(arrs, block, lambda *a, **kw: local_eval(*a, ev_pair=ev_pair, ev_near=ev_near, **kw))

    for _ in range(W):
        flush.zero_()
        step()
    torch.cuda.synchronize(dev)

    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    evp = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    evn = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    for a, b in evp + evn:  # torch creates the CUDA event lazily on first record: materialize the handles
        a.record(stream)
        b.record(stream)
    # 1 GPU: capture the evaluation once (the library only enqueues: no host sync, no allocation) and time
    # replays, so a small step's kernels are not spaced out by the Python + ctypes enqueue of each call;
    # the graph holds one pair of kernel events, read after each replay
    graph = None
    if world == 1 and args.graph != "off":
        torch.cuda.synchronize(dev)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            step(evp[0], evn[0])
        torch.cuda.synchronize(dev)
        graph.replay()  # a first replay outside the timed region
        torch.cuda.synchronize(dev)
    g_pair, g_near = [], []
    with ClockSampler(local) as clk:
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        for i in range(K):
            flush.zero_()  # L2 flush, outside the timed events
            ev[i][0].record(stream)
            if graph is not None:
                graph.replay()
                res_u, res_v = out_u, out_v
            else:
                res_u, res_v = step(evp[i], evn[i])
            ev[i][1].record(stream)
            if graph is not None:  # this replay's kernel events (the host sync is outside the timed events)
                torch.cuda.synchronize(dev)
                g_pair.append(evp[0][0].elapsed_time(evp[0][1]))
                g_near.append(evn[0][0].elapsed_time(evn[0][1]) if (nodes or not fused) else 0.0)
        torch.cuda.synchronize(dev)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        def agree(flag):  # any rank still short of samples -> every rank pads one more step
            if dist is None:
                return flag
            t = torch.tensor([1.0 if flag else 0.0], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            return bool(t.item() > 0)
        clk.pad(lambda: (step(), torch.cuda.synchronize(dev)), agree=agree)
    step_ms = [a.elapsed_time(b) for a, b in ev]
    pair_ms = g_pair if graph is not None else [a.elapsed_time(b) for a, b in evp]
    near_ms = g_near if graph is not None else [a.elapsed_time(b) for a, b in evn]
    total_s = max_over_ranks(sum(step_ms) / 1e3, dev)
    value = pairs * K / total_s
    u_host, v_host = res_u.cpu().numpy(), res_v.cpu().numpy()

    # end to end through the public API with pinned HOST buffers (copies inside the timed region):
    # N = 1: stokes_er_eval_host (H2D, evaluate, D2H in the library); N > 1: H2D of the inputs,
    # evaluate_sharded (incl. the all-gather), D2H of the gathered u, v
    e2e = None
    if not args.no_e2e:
        host = [torch.from_numpy(a).pin_memory() for a in block.arrays()]
        hu = torch.empty((3, M), dtype=torch.float64).pin_memory()
        hv = torch.empty((3, M), dtype=torch.float64).pin_memory()
        if nodes and world > 1:
            host = host[:5]  # the targets are the nodes: only the source arrays travel

            def e_step():
                d = [t.to(dev, non_blocking=True) for t in host]
                uu, vv = nodes_sharded_step(d, block, opt, ws, stream)
                hu.copy_(uu, non_blocking=True)
                hv.copy_(vv, non_blocking=True)
        elif nodes:
            host = host[:5]  # the targets are the nodes: only the source arrays travel
            hws = torch.empty(int(L.stokes_er_nodes_host_workspace_bytes(N, 3)), dtype=torch.uint8, device=dev)
            e_step = lambda: ser.evaluate_nodes_host(*host, block.h, block.rho, out_u=hu, out_v=hv, workspace=hws,
                                                     stream=stream)
        elif world == 1:
            hws = ser.alloc_workspace(M, N, 3, dev, host=True)
            e_step = lambda: ser.evaluate_host(*host, block.h, block.rho, out_u=hu, out_v=hv, workspace=hws,
                                               stream=stream)
        else:
            def e_step():
                d = [t.to(dev, non_blocking=True) for t in host]
                uu, vv = sharded_step(d, block, local_eval)
                hu.copy_(uu, non_blocking=True)
                hv.copy_(vv, non_blocking=True)
        for _ in range(2):
            e_step()
        torch.cuda.synchronize(dev)
        ke = max(3, K // 4)
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize(dev)
        e_ms = []
        for _ in range(ke):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            e_step()
            b.record(stream)
            b.synchronize()
            e_ms.append(a.elapsed_time(b))
        e_total = max_over_ranks(sum(e_ms) / 1e3, dev)
        e2e = {"value": pairs * ke / e_total, "unit": UNIT,
               "h2d_bytes_per_step": int(sum(t.numel() * t.element_size() for t in host)),
               "d2h_bytes_per_step": int(hu.numel() * 8 + hv.numel() * 8),
               "api": ("host->device copies + sharding.evaluate_nodes_sharded (all-reduce) + device->host copy"
                       if nodes and world > 1 else
                       "stokes_er_eval_nodes_host (C ABI, pinned host buffers)" if nodes else
                       "stokes_er_eval_host (C ABI, pinned host buffers)" if world == 1 else
                       "host->device copies + sharding.evaluate_sharded (all-gather) + device->host copy")}

    sol_err = solve_parity(block, dev, stream) if rank == 0 else None
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None

    near = near_pair_count(block)
    clocks = clk.summary()
    far_avg_s = statistics.mean(pair_ms) / 1e3
    far = pairs - near
    # per-rank kernel work: the local target range's share (Morton ranges: near pairs ~ uniform), or the
    # rank's 1/world of the node path's block-pair items
    share = (1.0 / world) if nodes else M_loc / M
    f_clk = 1965.0
    peak = SMS * FP64_LANES_PER_SM * 2 * f_clk * 1e6 / 1e12  # TFLOP/s
    peak_source = ("derived: 148 SMs x 64 FP64 FMA/clk/SM x 2 x 1965 MHz max SM clock (MEASURED_PEAKS.json has "
                   "no FP64 entry; DFMA-loop probe 34.2 TFLOP/s = 92% of it, tools/probes)")
    sym_pairs = nbr_pairs = None
    if nodes:
        sym_pairs, nbr_pairs = ser.nodes_pair_counts(N, block.h, block.rho, ws, stream=stream)
    if nodes:
        k_flops = sym_pairs / 2 * F_SYM_UNORDERED_ALG * share
        k_issued = sym_pairs / 2 * F_SYM_UNORDERED_ISSUED * share
        kname = ("sym_kernel<3> (FP64 pipe): the far-field sum (PAPER.md:183-191) over all-far 96-node block "
                 "pairs, one evaluation of each pair's shared part for both directed pairs (node targets)")
        kprefix = "void ser::sym_kernel<3>"
        conv = (f"{F_SYM_UNORDERED_ALG} algorithmic flops per unordered far pair = {F_SYM_UNORDERED_ALG / 2} per "
                "directed pair (rsqrt = 1, FMA = 2; the shared geometry and d.(q_j - q_i) counted once)")
    elif fused:
        k_flops = (far * F_FAR_ALG + near * F_NEAR_ALG) * share
        k_issued = (far * F_FAR_ISSUED + near * F_NEAR_ISSUED) * share
        kname = ("fused_kernel<3,T> (FP64 pipe): far-field sum (PAPER.md:183-191) + near 3-delta sums "
                 "with the folded extrapolation (PAPER.md:82-123), one persistent kernel")
        kprefix = "void ser::fused_kernel<3"
        conv = (f"{F_FAR_ALG} algorithmic flops per far pair + {F_NEAR_ALG} per near pair "
                "(rsqrt/erf/exp = 1, FMA = 2)")
    else:
        k_flops = far * F_FAR_ALG * share
        k_issued = far * F_FAR_ISSUED * share
        kname = "far_kernel<3,T> (FP64 pipe): the shared far-field sum, PAPER.md:183-191"
        kprefix = "void ser::far_kernel<3"
        conv = f"{F_FAR_ALG} algorithmic flops per far pair (rsqrt = 1, FMA = 2)"
    achieved = k_flops / far_avg_s / 1e12
    bench_cfg = {"workload": block.name, "path": "stokes_er_eval_nodes" if nodes else "stokes_er_eval",
                 "schedule": "nodes" if nodes else args.schedule, "targets_per_thread": int(opt.stats[3])}
    roofline = {"bound": "alu", "achieved": achieved, "peak": peak, "unit": "TFLOP/s", "frac": achieved / peak,
                "traffic": None, "traffic_source": "no ncu --set full capture of this exact configuration committed",
                "kernel": kname, "peak_source": peak_source,
                "flops_per_launch": k_flops, "flop_convention": conv,
                "frac_issued_convention": k_issued / far_avg_s / 1e12 / peak,
                "kernel_ms": far_avg_s * 1e3, "kernel_share": sum(pair_ms) / sum(step_ms),
                "timing": "CUDA events recorded by the library around the kernel on the launching stream"
                          + (" (inside the captured graph, read after each replay)" if graph is not None else ""),
                "far_pairs": far, "near_pairs": near}
    traffic = committed_traffic(bench_cfg, kprefix)
    if traffic:
        roofline["traffic"], roofline["traffic_source"] = traffic
    if clocks.get("sm_mhz"):
        roofline["frac_at_measured_clock"] = achieved / (SMS * FP64_LANES_PER_SM * 2 * clocks["sm_mhz"] / 1e6)
    near_info = None
    if nodes:
        near_avg_s = statistics.mean(near_ms) / 1e3
        roofline["far_pairs_per_s"] = sym_pairs * share / far_avg_s
        roofline["frac_57_flop_convention"] = sym_pairs * share * F_FAR_ALG / far_avg_s / 1e12 / peak
        roofline["directed_pairs"] = sym_pairs
        nbr_far = nbr_pairs - near
        near_info = {"kernel": "nbr_kernel<3>: near 3-delta pairs + the far pairs of the block pairs the "
                               "symmetric kernel leaves out (own block, not all-far)",
                     "ms": near_avg_s * 1e3, "share": sum(near_ms) / sum(step_ms), "pairs": nbr_pairs,
                     "near_pairs": near, "far_pairs": nbr_far,
                     "tflops_alg": (near * F_NEAR_ALG + nbr_far * F_FAR_ALG) / near_avg_s / 1e12}
    elif not fused:
        near_avg_s = statistics.mean(near_ms) / 1e3
        roofline["far_pairs_per_s"] = far * share / far_avg_s
        near_info = {"kernel": "near_kernel<3>", "ms": near_avg_s * 1e3, "share": sum(near_ms) / sum(step_ms),
                     "near_pairs": near, "near_pairs_per_s": near * share / near_avg_s,
                     "tflops_alg": near * share * F_NEAR_ALG / near_avg_s / 1e12}
    alg_flops = far * F_FAR_ALG + near * F_NEAR_ALG
    parity, def_s, def_pairs = sampled_parity(block, u_host, v_host)
    parity["solve_max_rel"] = sol_err
    parity["solve_tolerance"] = 1e-13
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
            "ms_per_step": 1e3 * total_s / K, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": {"workload": block.name, "N": N, "M": M, "pairs_per_step": pairs, "near_pairs_per_step": near,
                       "h": block.h, "rho": list(block.rho), "mode": "SL+DL", "cutoff": 6.0,
                       "l2": "flushed between timed steps (256 MiB write); inputs are larger than L2 at N >= 1e6",
                       "inputs": "resident in HBM", "seed": block.meta.get("seed"),
                       "targets_per_thread": int(opt.stats[3]), "work_items": int(opt.stats[0]),
                       "grid_ctas": int(opt.stats[1]), "chunk_tiles": int(opt.stats[2]),
                       "schedule": "nodes" if nodes else args.schedule,
                       "path": "stokes_er_eval_nodes" if nodes else "stokes_er_eval",
                       "launch": ("CUDA-graph replay of one evaluation (captured once after the warm-up; the "
                                  "library's kernels, timed by events on the replay stream)" if graph is not None
                                  else "eager (one C-ABI call per step)"),
                       "parallelism": ("single GPU" if world == 1 else
                                       f"node-path shards x{world}: 1/{world} of the symmetric kernel's block-pair "
                                       "items and of the neighbour units per rank (sharding.evaluate_nodes_sharded), "
                                       "all-reduce of u, v in the timed region" if nodes else
                                       f"target-sharded x{world}: Morton ranges of ONE target set "
                                       "(sharding.evaluate_sharded), sources replicated, all-gather of u, v in the "
                                       "timed region")},
            "fp64_tflops_alg": alg_flops * K / total_s / 1e12,
            "fp64_tflops_alg_note": "whole step, SURVEY 8(d) per-pair convention: 57 flops per far pair + 180 per "
                                    "near pair, every directed pair counted",
            "roofline": roofline, "clocks": clocks, "parity": parity,
            "gpu_launches": K * (ser.nodes_launch_count(N, 3) if nodes else
                                 ser.launch_count(M_loc, N, 3) + (0 if fused else 1)),
            "gpu_launches_note": ("our kernels per step: bbox, morton, pack_sources, pack_node_soa, block_boxes, "
                                  "sym_kernel, nbr_kernel, finalize_nodes (+ CUB radix-sort launches, library code)"
                                  if nodes else
                                  ("our kernels per step and rank: small_rank, pack_both, "
                                   if ser.launch_count(M_loc, N, 3) == 4 else
                                   "our kernels per step and rank: bbox, 2 morton, pack_sources, pack_targets, ")
                                  + ("fused far+near" if fused else "far, near") + ", finalize"
                                  + ("" if ser.launch_count(M_loc, N, 3) == 4 else
                                     " (+ CUB radix-sort launches, library code)")),
            "e2e": e2e}
    if near_info is not None:
        line["near_kernel"] = near_info
    if not args.no_cpu_baseline and world == 1:
        line["cpu_baseline"] = cpu_baseline(block, definition=(def_s, def_pairs))
    if dist is not None:
        dist.destroy_process_group()
    return line



def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))

    if args.impl == "reference":
        line = run_reference(args, rank, world)
    elif args.workload == "tree":
        line = run_tree(args, rank, world)
    elif args.workload == "onsurface":
        line = run_onsurface(args, rank, world)
    elif args.workload == "twodrop":
        line = run_twodrop(args, rank, world)
    elif args.config == 4:
        line = run_config4(args, rank, world)
    else:
        line = run_eval(args, rank, world)
    if line is not None:
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()

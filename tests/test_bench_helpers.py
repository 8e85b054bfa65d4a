"""Host-side helpers of bench.py and the node-target input helper (CPU only)."""
from __future__ import annotations

import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_committed_traffic_only_for_the_same_bench_configuration(tmp_path, monkeypatch):
    """roofline.traffic comes from an ncu summary only if its recorded bench configuration
    (workload, path, schedule, targets per thread) equals the run's; otherwise None."""
    import bench

    cfg = {"workload": "cfg5_sphere_h1/256", "path": "stokes_er_eval_nodes", "schedule": "nodes",
           "targets_per_thread": 2}
    d = tmp_path / "profiles" / "r99"
    d.mkdir(parents=True)
    doc = {"bench_config": cfg, "kernels": [{"kernel": "void sym_kernel<3>(SymParams)",  # as ncu names it
                                             "dram__bytes_read.sum": "1.5 Gbyte",
                                             "dram__bytes_write.sum": "250 Mbyte"}]}
    (d / "ncu_full_test.json").write_text(json.dumps(doc))
    monkeypatch.setattr(bench, "ROOT", str(tmp_path))
    got = bench.committed_traffic(cfg, "void ser::sym_kernel<3>")
    assert got is not None and got[0] == int(1.75e9) and "ncu_full_test.json" in got[1]
    for key, other in (("workload", "cfg5_sphere_h1/128"), ("path", "stokes_er_eval"), ("schedule", "fused"),
                       ("targets_per_thread", 1)):
        assert bench.committed_traffic(dict(cfg, **{key: other}), "void ser::sym_kernel<3>") is None
    assert bench.committed_traffic(cfg, "void ser::fused_kernel<3") is None  # another kernel


def test_node_block_is_the_node_target_argument_set():
    """workloads.configs.node_block: targets = the nodes, b = 0, x0 density rows = (n, f, q) at the
    nodes -- what stokes_er_eval_nodes computes; config 5 is already that block."""
    from workloads.configs import config3, config5, node_block

    c5 = config5(inv_h=8)
    nb = node_block(c5)
    for a, b in zip(c5.arrays(), nb.arrays()):
        np.testing.assert_array_equal(a, b)
    e = node_block(config3(inv_h=8))
    assert e.M == e.N and np.all(e.tgt_b == 0.0)
    np.testing.assert_array_equal(e.tgt_xyz, e.src_xyz)
    np.testing.assert_array_equal(e.tgt_x0_density, np.concatenate([e.src_normal, e.f, e.q]))

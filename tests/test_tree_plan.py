"""NEXT-3 host logic on CPU (-m "not gpu"): stokes_er_tree_build is plain host C++
in libstokes_er.so, so the octree the GPU path uses is checked here against the
reading R22 and against the oracle's own tree (node counts), without a GPU."""
from __future__ import annotations

import ctypes

import numpy as np
import pytest

import oracle
from workloads.configs import config2, config3

NODE = np.dtype([("lo", "<f8", 3), ("hi", "<f8", 3), ("c", "<f8", 3), ("rc", "<f8"), ("begin", "<i4"),
                 ("end", "<i4"), ("first_child", "<i4"), ("nchild", "<i4"), ("level", "<i4"), ("pad", "<i4")])
HDR = np.dtype([("magic", "<u8"), ("N", "<i8"), ("nnodes", "<i4"), ("max_nodes", "<i4"), ("leaf_size", "<i4"),
                ("depth", "<i4"), ("off_nodes", "<i8"), ("off_perm", "<i8")])


def parse(plan):
    h = np.frombuffer(plan.buf, dtype=HDR, count=1)[0]
    nodes = np.frombuffer(plan.buf, dtype=NODE, count=int(h["nnodes"]), offset=int(h["off_nodes"]))
    perm = np.frombuffer(plan.buf, dtype="<i4", count=int(h["N"]), offset=int(h["off_perm"]))
    return h, nodes, perm


@pytest.fixture(scope="module")
def ser():
    import paper_2507_00156_b200 as ser

    ser._lib.load()
    return ser


@pytest.mark.parametrize("N0", [64, 300, 2000])
def test_tree_invariants(ser, N0):
    blk = config3(inv_h=32)
    x = blk.src_xyz
    plan = ser.TreePlan(x, N0, 6, 0.6)
    h, nodes, perm = parse(plan)
    assert h["N"] == x.shape[1] and h["nnodes"] == plan.nodes
    assert np.array_equal(np.sort(perm), np.arange(x.shape[1]))  # a permutation
    assert nodes[0]["begin"] == 0 and nodes[0]["end"] == x.shape[1]
    for nd in nodes:
        pts = x[:, perm[nd["begin"]:nd["end"]]]
        np.testing.assert_array_equal(nd["lo"], pts.min(axis=1))  # tight boxes (R22)
        np.testing.assert_array_equal(nd["hi"], pts.max(axis=1))
        assert nd["rc"] == pytest.approx(0.5 * np.linalg.norm(nd["hi"] - nd["lo"]), rel=1e-15)
        if nd["nchild"] == 0:
            assert nd["end"] - nd["begin"] <= N0 or np.all(nd["hi"] == nd["lo"])
        else:
            ch = nodes[nd["first_child"]:nd["first_child"] + nd["nchild"]]
            assert ch[0]["begin"] == nd["begin"] and ch[-1]["end"] == nd["end"]
            assert np.all(ch["begin"][1:] == ch["end"][:-1])  # children partition the parent
            assert np.all(ch["level"] == nd["level"] + 1)
            mid = 0.5 * (nd["lo"] + nd["hi"])
            for c in ch:  # every child sits in one octant of the parent's midpoint split
                pts = x[:, perm[c["begin"]:c["end"]]]
                up = pts >= mid[:, None]
                assert np.all(up.all(axis=1) | (~up).all(axis=1))


@pytest.mark.parametrize("N0", [200, 500, 2000])
def test_tree_matches_oracle_node_count(ser, oracle_mod, N0):
    """The library's tree and the oracle's independently built tree (R22) have the same size."""
    blk = config2(inv_h=32)
    plan = ser.TreePlan(blk.src_xyz, N0, 4, 0.6)
    _, _, st = oracle_mod.evaluate_tree_block(blk.take_targets(np.arange(3)), leaf_size=N0, degree=4, theta=0.6,
                                              stats=True)
    assert plan.nodes == st[0]


def test_tree_plan_errors(ser):
    x = config2(inv_h=16).src_xyz
    with pytest.raises(ValueError):
        ser.TreePlan(x, 0, 6, 0.6)        # leaf size < 1
    with pytest.raises(ValueError):
        ser.TreePlan(x, 100, 17, 0.6)     # degree > 16
    with pytest.raises(ValueError):
        ser.TreePlan(x, 100, 6, -1.0)     # theta < 0
    bad = x.copy()
    bad[0, 5] = np.nan
    with pytest.raises(ser._lib.StokesERError):
        ser.TreePlan(bad, 100, 6, 0.6)    # non-finite node
    L = ser._lib.load()
    p = ser._lib.TreeParams(100, 6, 0.6)
    assert L.stokes_er_tree_build(None, 10, ctypes.byref(p), None, 0) == 1  # EINVAL

"""NEXT-3 GPU parity (-m gpu): stokes_er_eval_tree against the treecode oracle
(oracle_eval_tree, the paper's per-target traversal, Sec. 3.4) on the
same seeded inputs.  Both sides build the same tree (R22), make the same MAC
and guard decisions (R23, plain FP64) and use the same Chebyshev modified
weights (R24), so they agree to rounding: max-norm relative <= 1e-12.
"""
from __future__ import annotations

import numpy as np
import pytest

import oracle
from workloads.configs import config1, config2, config5

pytestmark = pytest.mark.gpu
TOL = 1e-12


@pytest.fixture(scope="module")
def ser():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("CUDA device required for -m gpu tests")
    import paper_2507_00156_b200 as ser

    ser._lib.load()
    return ser


def rel(a, b):
    return float(np.abs(np.asarray(a) - np.asarray(b)).max() / np.abs(np.asarray(b)).max())


def check(ser, blk, mode=3, **tp):
    u, v = ser.evaluate_tree_block(blk, mode=mode, **tp)
    ur, vr = oracle.evaluate_tree_block(blk, mode=mode, **tp)
    if mode & 1:
        assert rel(u.cpu().numpy(), ur) <= TOL
    if mode & 2:
        assert rel(v.cpu().numpy(), vr) <= TOL
    return u, v


@pytest.mark.parametrize("tp", [dict(leaf_size=200, degree=4, theta=0.6), dict(leaf_size=500, degree=6, theta=0.6),
                                dict(leaf_size=300, degree=8, theta=0.4), dict(leaf_size=1000, degree=10, theta=0.8)])
def test_tree_parity_config2(ser, tp):
    blk = config2(inv_h=32)
    check(ser, blk.take_targets(np.arange(0, blk.M, 9)), **tp)


@pytest.mark.parametrize("mode", [1, 2])
def test_tree_parity_single_modes(ser, mode):
    blk = config2(inv_h=32)
    check(ser, blk.take_targets(np.arange(0, blk.M, 11)), mode=mode, leaf_size=400, degree=6, theta=0.6)


def test_tree_parity_near_targets(ser):
    """Config 1 (b/h in {0, +-1, +-2, +-3}): near pairs in directly summed leaves."""
    check(ser, config1(inv_h=16), leaf_size=300, degree=8, theta=0.6)


def test_theta_zero_equals_direct(ser):
    """theta = 0: the MAC never holds, every leaf is summed directly: the direct path's result."""
    blk = config2(inv_h=32)
    sub = blk.take_targets(np.arange(0, blk.M, 7))
    u, v = ser.evaluate_tree_block(sub, leaf_size=500, degree=4, theta=0.0)
    ud, vd = ser.evaluate_block(sub)
    assert rel(u.cpu().numpy(), ud.cpu().numpy()) <= 1e-13 and rel(v.cpu().numpy(), vd.cpu().numpy()) <= 1e-13


def test_tree_policy_config5_h64_sampled(ser):
    """The paper's parameter policy at h = 1/64 (eq. (33): theta 0.6, N0 2000, p 6), all
    N targets on the GPU; 257 sampled targets against the oracle."""
    blk = config5(inv_h=64)
    u, v = ser.evaluate_tree_block(blk, leaf_size=2000, degree=6, theta=0.6)
    idx = np.unique(np.concatenate([np.arange(0, blk.M, blk.M // 256), [blk.M - 1]]))
    ur, vr = oracle.evaluate_tree_block(blk.take_targets(idx), leaf_size=2000, degree=6, theta=0.6)
    assert rel(u.cpu().numpy()[:, idx], ur) <= TOL and rel(v.cpu().numpy()[:, idx], vr) <= TOL


def test_tree_plan_reuse_and_errors(ser):
    import torch

    blk = config2(inv_h=16)
    plan = ser.TreePlan(blk.src_xyz, 300, 6, 0.6)
    arrs = ser.to_device(blk)
    a = ser.evaluate_tree(*arrs, blk.h, blk.rho, plan)
    b = ser.evaluate_tree(*arrs, blk.h, blk.rho, plan)
    assert torch.equal(a[0], b[0]) and torch.equal(a[1], b[1])  # deterministic, plan reusable
    with pytest.raises(ValueError):
        ser.TreePlan(blk.src_xyz, 300, 40, 0.6)  # degree > 16
    other = ser.TreePlan(blk.src_xyz[:, :100], 300, 6, 0.6)
    with pytest.raises(ValueError):
        ser.evaluate_tree(*arrs, blk.h, blk.rho, other)


def test_tree_onsurface_parity(ser):
    """NEXT-1 s# with the treecode far part (config 5 at 1/h = 64, delta = 3h, cutoff 7):
    against oracle_eval_tree_sharp on sampled targets, and theta = 0 against the direct s# path."""
    blk = config5(inv_h=64)
    d = 3 * blk.h
    plan = ser.TreePlan(blk.src_xyz, 2000, 6, 0.6)
    arrs = ser.to_device(blk)
    u, v = ser.evaluate_tree_onsurface(*arrs, d, plan)
    idx = np.arange(0, blk.M, 263)
    sub = blk.take_targets(idx)
    ur, vr = oracle.evaluate_tree_sharp(*sub.arrays(), d, leaf_size=2000, degree=6, theta=0.6)
    assert rel(u.cpu().numpy()[:, idx], ur) <= TOL and rel(v.cpu().numpy()[:, idx], vr) <= TOL
    plan0 = ser.TreePlan(blk.src_xyz, 2000, 6, 0.0)
    u0, v0 = ser.evaluate_tree_onsurface(*arrs, d, plan0)
    ud, vd = ser.evaluate_onsurface(*arrs, d)
    assert rel(u0.cpu().numpy(), ud.cpu().numpy()) <= 1e-13 and rel(v0.cpu().numpy(), vd.cpu().numpy()) <= 1e-13

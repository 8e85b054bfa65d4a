"""NEXT-3 pins (CPU, -m "not gpu"): the treecode oracle (Sec. 3.4, lines
194-233; readings R22-R25 in oracle/stokes_er_oracle.c) against the direct
localized sum, which the C oracle already pins to closed forms and mpmath.

  * theta = 0 (the MAC never holds) and N0 >= N (one leaf) reduce the treecode
    to the direct localized sum exactly (every source in exactly one leaf)
  * the far approximation (eqs. (29)-(32)) converges to the direct sum
    geometrically in the degree p (a wrong kernel, sign, channel or weight
    would stall it), and more strictly for smaller theta
  * accepted clusters never contain near pairs (R23): results are unchanged
    whichever near targets are included
  * R26: accepted clusters with at most (p+1)^3 points are summed directly, so
    a degree so high that every cluster is "small" gives the direct sum
"""
from __future__ import annotations

import numpy as np
import pytest

from workloads.configs import config1, config2


@pytest.fixture(scope="module")
def cfg2_sub():
    blk = config2(inv_h=32)
    return blk.take_targets(np.arange(0, blk.M, 25))


@pytest.fixture(scope="module")
def direct(oracle_mod, cfg2_sub):
    return oracle_mod.evaluate_block(cfg2_sub, localized=True)


def rel(a, b):
    return float(np.abs(a - b).max() / np.abs(b).max())


def test_theta_zero_is_the_direct_sum(oracle_mod, cfg2_sub, direct):
    u, v, st = oracle_mod.evaluate_tree_block(cfg2_sub, leaf_size=200, degree=4, theta=0.0, stats=True)
    assert st[1] == 0 and st[2] == cfg2_sub.M * cfg2_sub.N
    assert rel(u, direct[0]) <= 1e-15 and rel(v, direct[1]) <= 1e-15


def test_single_leaf_is_the_direct_sum(oracle_mod, cfg2_sub, direct):
    u, v, st = oracle_mod.evaluate_tree_block(cfg2_sub, leaf_size=10 ** 7, degree=6, theta=0.6, stats=True)
    assert st[0] == 1
    assert rel(u, direct[0]) <= 1e-15 and rel(v, direct[1]) <= 1e-15


def test_degree_convergence(oracle_mod, cfg2_sub, direct):
    """theta = 0.6: error vs direct falls by > 10x per +2 in p."""
    errs = []
    for p in (4, 6, 8, 10):
        u, v, st = oracle_mod.evaluate_tree_block(cfg2_sub, leaf_size=500, degree=p, theta=0.6, stats=True)
        assert st[1] > 0 and st[2] < 0.8 * cfg2_sub.M * cfg2_sub.N  # the approximation is in use
        errs.append(max(rel(u, direct[0]), rel(v, direct[1])))
    for a, b in zip(errs, errs[1:]):
        assert b < a / 10.0, errs
    assert errs[-1] < 1e-8


def test_smaller_theta_is_more_accurate(oracle_mod, cfg2_sub, direct):
    e = {}
    for th in (0.4, 0.6, 0.8):
        u, v = oracle_mod.evaluate_tree_block(cfg2_sub, leaf_size=500, degree=6, theta=th)
        e[th] = max(rel(u, direct[0]), rel(v, direct[1]))
    assert e[0.4] < e[0.6] < e[0.8]


def test_near_targets_match_direct_regularization(oracle_mod):
    """Config-1 targets at b/h in {0, +-1, +-2, +-3}: the treecode keeps every near pair
    in a directly summed leaf, so with p = 10 the extrapolated values agree with the
    direct method to the far approximation's accuracy (not to the O(1)
    regularization difference an approximated near pair would cause)."""
    blk = config1(inv_h=16, per_class=6)
    ud, vd = oracle_mod.evaluate_block(blk, localized=True)
    u, v = oracle_mod.evaluate_tree_block(blk, leaf_size=300, degree=10, theta=0.6)
    assert rel(u, ud) < 1e-8 and rel(v, vd) < 1e-8


def test_small_clusters_summed_directly(oracle_mod, cfg2_sub, direct):
    """R26: with (p+1)^3 >= N every accepted cluster is summed directly: the direct sum."""
    u, v, st = oracle_mod.evaluate_tree_block(cfg2_sub, leaf_size=500, degree=26, theta=0.6, stats=True)
    assert st[1] == 0 and st[2] == cfg2_sub.M * cfg2_sub.N
    assert rel(u, direct[0]) <= 1e-14 and rel(v, direct[1]) <= 1e-14

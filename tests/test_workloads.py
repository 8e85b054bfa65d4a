"""Pins of the seeded input generator (CPU only)."""
from __future__ import annotations

import json
import math
import os

import numpy as np
import pytest

from workloads.configs import config1, config2, config3, config4, config5, subsample
from workloads.quadrature import (Ellipsoid, bump, grid_targets_outside, partition_of_unity, quadrature,
                                  sphere)

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_counts.json")))


@pytest.mark.parametrize("row", GOLDEN["rows"], ids=lambda r: f"1/h={r['inv_h']}")
def test_table1_quadrature_counts(row):
    """PAPER.md Table 1 '# quads' (lines 266-272) for the spheroid of PAPER.md:245."""
    x, n, w, _ = quadrature(Ellipsoid(tuple(GOLDEN["surface_axes"])), 1.0 / row["inv_h"])
    assert x.shape[1] == row["quads"]


@pytest.mark.parametrize("row", GOLDEN["rows"][:3], ids=lambda r: f"1/h={r['inv_h']}")
def test_table1_target_counts(row):
    """PAPER.md Table 1 '# targets': grid points outside, within distance h,
    read as 0 <= b <= h (R13)."""
    h = 1.0 / row["inv_h"]
    y, x0, b = grid_targets_outside(Ellipsoid(tuple(GOLDEN["surface_axes"])), h, h)
    assert y.shape[1] == row["targets"]


def test_bump_and_partition_of_unity():
    """PAPER.md:152-159."""
    assert bump(0.0) == 1.0
    assert bump(0.5) == pytest.approx(math.exp(-2.0 / 3.0), rel=1e-15)
    assert bump(1.0) == 0.0 and bump(-1.2) == 0.0
    rng = np.random.default_rng(0)
    n = rng.standard_normal((3, 10000))
    n /= np.linalg.norm(n, axis=0)
    psi = partition_of_unity(n)
    assert np.abs(psi.sum(axis=0) - 1).max() < 1e-14
    assert psi.min() >= 0 and psi.max() <= 1
    np.testing.assert_allclose(partition_of_unity(np.array([[1.0], [0.0], [0.0]]))[:, 0], [1, 0, 0])
    s = 1 / math.sqrt(3)
    np.testing.assert_allclose(partition_of_unity(np.array([[s], [s], [s]]))[:, 0], [1 / 3] * 3, atol=1e-15)


def test_sphere_area_converges():
    """The rule is high order: area error 4.1e-5 at 1/16, -7.1e-7 at 1/32."""
    errs = []
    for inv in (16, 32, 64):
        x, n, w, _ = quadrature(sphere(), 1.0 / inv)
        errs.append(abs(w.sum() - 4 * math.pi))
    assert errs[0] < 5e-5 and errs[1] < 1e-6 and errs[2] < 1e-8
    x, n, w, _ = quadrature(sphere(), 1 / 32)
    assert (w >= 0).all()  # nodes at the angular cutoff carry psi ~ 0 (bump underflow)
    np.testing.assert_allclose(np.linalg.norm(n, axis=0), 1, atol=1e-15)
    np.testing.assert_allclose(np.linalg.norm(x, axis=0), 1, atol=1e-15)


def test_config_shapes_and_consistency():
    b1 = config1()
    assert (b1.N, b1.M) == (4302, 504)
    b2 = config2(inv_h=32)
    assert (b2.N, b2.M) == (17070, 17070 + 8535)
    for blk in (b1, b2, config3(inv_h=32)):
        # y = x0 + b n0 and |n0| = 1 (inputs trusted by the library, include/stokes_er.h)
        n0 = blk.tgt_x0_density[:3]
        np.testing.assert_allclose(np.linalg.norm(n0, axis=0), 1, atol=1e-14)
        np.testing.assert_allclose(blk.tgt_xyz, blk.tgt_x0 + blk.tgt_b * n0, atol=1e-14)
        for a in blk.arrays():
            assert a.dtype == np.float64 and a.flags.c_contiguous
    # seeded: same seed, same arrays
    np.testing.assert_array_equal(config1().f, config1().f)
    assert not np.array_equal(config1(seed=2).f, config1().f)


def test_config4_blocks():
    blocks = config4(eps=0.1, inv_h=16)
    assert [b.name.split("_")[-1] for b in blocks] == ["A<-A", "A<-B", "B<-A", "B<-B"]
    cross = blocks[1]
    assert cross.tgt_b.min() >= 0.1 - 1e-12  # gap eps
    assert blocks[0].N == blocks[3].N


def test_config5_and_subsample():
    b5 = config5(inv_h=32)
    assert b5.M == b5.N == 17070
    s = subsample(b5, 100)
    assert s.M == 100 and s.N == b5.N

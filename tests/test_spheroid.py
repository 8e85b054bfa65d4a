"""PAPER.md Table 1 (lines 262-274) reproduced by the oracle (-m "not gpu") and by the
GPU path (-m gpu): the Stokeslet integral at grid points within h outside the translating
prolate spheroid, against the exact velocity (tests/closed_forms.py, Chwang & Wu's
singularity solution), max and L2 errors as the paper prints them (3 significant digits).
This pins the whole method -- quadrature, subtraction, regularization, localization and
the extrapolation with rho = (3,4,5) -- to the paper's own printed numbers."""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from closed_forms import spheroid_translation_velocity
from workloads.quadrature import Ellipsoid, quadrature
from workloads.spheroid import AXES, spheroid_block, traction

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "table1_errors.json")))["rows"]


def errors(u, y):
    e = np.linalg.norm(u - spheroid_translation_velocity(y), axis=0)
    return float(e.max()), float(np.sqrt((e ** 2).mean()))


def test_exact_velocity_is_the_rigid_motion_on_the_surface():
    x, _, _, _ = quadrature(Ellipsoid(AXES), 1.0 / 16)
    u = spheroid_translation_velocity(x[:, ::7])
    np.testing.assert_allclose(u, np.repeat([[1.0], [0.0], [0.0]], u.shape[1], axis=1), atol=1e-13)


def test_exact_velocity_matches_the_plain_single_layer_away_from_the_surface():
    """(1/8pi) sum S f w with the paper's quadrature at 1/h = 128 (spectrally accurate away
    from the surface) at the origin (inside: the translation velocity) and at exterior points."""
    x, _, w, _ = quadrature(Ellipsoid(AXES), 1.0 / 128)
    fw = traction(x) * w
    pts = np.array([[0.0, 0.0, 0.0], [1.4, 0.0, 0.0], [0.0, 0.9, 0.2], [0.6, 0.5, -0.5], [-1.2, 0.4, 0.3]]).T
    for t in range(pts.shape[1]):
        d = pts[:, t:t + 1] - x
        R = np.linalg.norm(d, axis=0)
        u = ((fw / R) + d * ((d * fw).sum(0) / R ** 3)).sum(1) / (8 * np.pi)
        ex = np.array([1.0, 0.0, 0.0]) if t == 0 else spheroid_translation_velocity(pts[:, t:t + 1])[:, 0]
        np.testing.assert_allclose(u, ex, atol=1e-8)


@pytest.mark.parametrize("inv_h", [32, 64])
def test_table1_errors_oracle(oracle_mod, inv_h):
    blk = spheroid_block(inv_h)
    g = GOLDEN[str(inv_h)]
    assert (blk.N, blk.M) == (g["quads"], g["targets"])
    u, _ = oracle_mod.evaluate_block(blk, mode=1, localized=True)
    mx, l2 = errors(u, blk.tgt_xyz)
    assert mx == pytest.approx(g["max_err"], rel=0.01) and l2 == pytest.approx(g["l2_err"], rel=0.01), (mx, l2)


@pytest.mark.gpu
@pytest.mark.parametrize("inv_h", [32, 64, 128, 256])
def test_table1_errors_gpu(inv_h):
    import paper_2507_00156_b200 as ser

    blk = spheroid_block(inv_h)
    u, _ = ser.evaluate_block(blk, mode=1)
    mx, l2 = errors(u.cpu().numpy(), blk.tgt_xyz)
    g = GOLDEN[str(inv_h)]
    assert mx == pytest.approx(g["max_err"], rel=0.01) and l2 == pytest.approx(g["l2_err"], rel=0.01), (mx, l2)

"""Pins of the CPU oracle against things other than itself (CPU only, -m "not gpu").

Each test names what fixes the expected value: a closed form, an exact
rational, a 50-digit mpmath evaluation, or a paper-printed number.
"""
from __future__ import annotations

import json
import os
from fractions import Fraction

import mpmath as mp
import numpy as np
import pytest

import hp  # noqa: E402
from pair_blocks import one_pair_block
from closed_forms import (SHEAR_TRACTION, SHEAR_VELOCITY, chi_of_b, sl_rotation, sl_translation)
from workloads.configs import config1, config2
from workloads.densities import ConstField, LinearField, RigidField, ZeroField

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


# ---------------------------------------------------------------- scalar pins
@pytest.mark.parametrize("t", [1e-6, 1e-3, 0.1, 0.5, 1.0, 1.7, 3.0, 4.5, 6.0, 9.0])
def test_s_factors_vs_mpmath(oracle_mod, t):
    """eqs. (14)-(16), against 50-digit mpmath.  Absolute
    error ~eps*t is the direct form's bound (R4)."""
    got = oracle_mod.s_factors(t)
    ref = [float(v) for v in hp.s_factors(t)]
    for g, r in zip(got, ref):
        assert abs(g - r) <= 4e-16 * max(1.0, t) ** 3
    assert abs(got[0] - ref[0]) <= 2e-16 * abs(ref[0])  # s1 = erf keeps relative accuracy


def test_s_factors_decay_at_cutoff(oracle_mod):
    """(1-s_i(t)) negligible for t > 6.  1 - s3(6) = 3.93e-14 (SURVEY 4.3 erratum 1)."""
    s = oracle_mod.s_factors(6.0)
    ref = [1 - hp.s_factors(6.0)[i] for i in range(3)]
    assert float(ref[2]) == pytest.approx(3.93e-14, rel=2e-3)
    for i in range(3):
        assert abs((1 - s[i]) - float(ref[i])) < 3e-16


@pytest.mark.parametrize("t", [0.25, 1.0, 2.5, 5.0])
def test_s_sharp_vs_mpmath(oracle_mod, t):
    """on-surface factors."""
    got = oracle_mod.s_sharp_factors(t)
    ref = [float(v) for v in hp.s_sharp(t)]
    np.testing.assert_allclose(got, ref, rtol=0, atol=2e-15 * max(1, t) ** 5)


@pytest.mark.parametrize("lam", [0.0, 0.25, -0.5, 0.75, 1.0, -1.5, 2.0, 3.0, 4.0])
def test_I0_I2_vs_mpmath(oracle_mod, lam):
    """eqs. (18)-(19); even in lambda by the |lambda|."""
    i0, i2 = oracle_mod.I0(lam), oracle_mod.I2(lam)
    r0, r2 = float(hp.I0(lam)), float(hp.I2(lam))
    cancel = 1.0 + 2.0 * lam * lam * (1 + lam * lam)  # FP64 cancellation factor of the direct formula
    assert abs(i0 - r0) <= 4e-16 * cancel * abs(r0) + 1e-300
    assert abs(i2 - r2) <= 4e-16 * cancel * (1 + lam ** 2) * abs(r2) + 1e-300


def test_I0_I2_at_zero_closed_form(oracle_mod):
    assert oracle_mod.I0(0.0) == pytest.approx(1 / np.sqrt(np.pi), rel=1e-15)
    assert oracle_mod.I2(0.0) == pytest.approx(1 / (3 * np.sqrt(np.pi)), rel=1e-15)


# ----------------------------------------------------------- extrapolation
def _weights(oracle_mod, b, h, rho):
    ind = np.zeros((3, 3, 1))
    for k in range(3):
        ind[k, k, 0] = 1.0
    return oracle_mod.extrapolate(np.array([b]), h, rho, ind)[:, 0]


def test_extrapolation_b0_exact_rationals(oracle_mod):
    """golden/extrapolation_b0.json: lambda = 0 weights are exact rationals."""
    cases = json.load(open(os.path.join(GOLDEN, "extrapolation_b0.json")))["cases"]
    for c in cases:
        w = _weights(oracle_mod, 0.0, 1 / 32, c["rho"])
        exact = [float(Fraction(s)) for s in c["weights"]]
        np.testing.assert_allclose(w, exact, rtol=0, atol=2e-14)


@pytest.mark.parametrize("b_over_h", [0.0, 0.5, -1.0, 2.0, 3.0, -5.5, 9.0])
def test_extrapolation_manufactured_round_trip(oracle_mod, b_over_h):
    """eq. (17): build u^dk = u + c1 rho I0 + c2 rho^3 I2 with 50-digit I0/I2,
    the solve must return u (SPEC.md:333 idea, values independent of the oracle)."""
    h, rho = 1 / 64, (2.0, 3.0, 4.0)
    b = b_over_h * h
    rng = np.random.default_rng(7)
    u = rng.uniform(-1, 1, 5)
    c1 = rng.uniform(-1, 1, 5)
    c2 = rng.uniform(-1, 1, 5)
    ind = np.zeros((3, 5, 1))
    for k, r in enumerate(rho):
        lam = mp.mpf(b) / (mp.mpf(r) * mp.mpf(h))
        for c in range(5):
            ind[k, c, 0] = float(mp.mpf(u[c]) + mp.mpf(c1[c]) * r * hp.I0(lam) + mp.mpf(c2[c]) * r ** 3 * hp.I2(lam))
    got = oracle_mod.extrapolate(np.array([b]), h, rho, ind)[:, 0]
    np.testing.assert_allclose(got, u, rtol=0, atol=5e-14)


def test_extrapolation_shift_and_constant(oracle_mod):
    """first column of A is all ones: adding kappa to all u^dk shifts u by kappa;
    equal u^dk return that value."""
    rng = np.random.default_rng(3)
    M = 64
    b = rng.uniform(-3, 3, M) / 32
    ind = rng.standard_normal((3, 2, M))
    base = oracle_mod.extrapolate(b, 1 / 32, (2, 3, 4), ind)
    shifted = oracle_mod.extrapolate(b, 1 / 32, (2, 3, 4), ind + 0.75)
    np.testing.assert_allclose(shifted - base, 0.75, rtol=0, atol=1e-13)
    const = np.repeat(ind[:1], 3, axis=0)
    np.testing.assert_allclose(oracle_mod.extrapolate(b, 1 / 32, (2, 3, 4), const), ind[0], rtol=0, atol=1e-13)


def test_extrapolation_far_target_passthrough(oracle_mod):
    """|b| >> delta: I0, I2 underflow, system singular -> u^d1 (reading R7)."""
    ind = np.random.default_rng(1).standard_normal((3, 3, 2))
    out = oracle_mod.extrapolate(np.array([3.0, -3.0]), 1 / 64, (2, 3, 4), ind)
    np.testing.assert_array_equal(out, ind[0])


def test_extrapolation_weights_sum_to_one(oracle_mod):
    for bh in np.linspace(-4, 4, 17):
        w = _weights(oracle_mod, bh / 32, 1 / 32, (2, 3, 4))
        assert abs(w.sum() - 1) < 1e-13
        # even in b (I0, I2 use |lambda|)
        np.testing.assert_allclose(w, _weights(oracle_mod, -bh / 32, 1 / 32, (2, 3, 4)), atol=1e-15)


# ------------------------------------------------------- closed-form sphere pins
F_T = np.array([1.0, 0.0, 0.0])
Q_C = np.array([1.0, -2.0, 0.5])
OMEGA = np.array([0.3, -0.5, 0.7])
RIGID = dict(U=(0.2, 0.1, -0.4), Omega=(1.0, 0.5, -0.25))


def _err(block, f_field, q_field, oracle_mod, localized=True):
    u, v = oracle_mod.evaluate_block(block, localized=localized)
    return u, v


@pytest.fixture(scope="module")
def sphere_runs(oracle_mod):
    """Config-1 targets (b/h in {0, +-1, +-2, +-3}) at 1/h = 16 and 32 for the closed-form fields."""
    out = {}
    for inv in (16, 32):
        runs = {}
        blk = config1(f_field=ConstField(F_T), q_field=ConstField(Q_C), inv_h=inv, per_class=24)
        runs["transl"] = (blk, *oracle_mod.evaluate_block(blk, localized=True))
        blk = config1(f_field=RigidField(Omega=OMEGA), q_field=RigidField(**RIGID), inv_h=inv, per_class=24)
        runs["rigid"] = (blk, *oracle_mod.evaluate_block(blk, localized=True))
        blk = config1(f_field=LinearField(SHEAR_TRACTION), q_field=LinearField(SHEAR_VELOCITY), inv_h=inv,
                      per_class=24)
        runs["shear"] = (blk, *oracle_mod.evaluate_block(blk, localized=True))
        out[inv] = runs
    return out


def _errors(runs):
    blk, u, v = runs["transl"]
    y = blk.tgt_xyz
    chi = chi_of_b(blk.tgt_b)
    e = {"sl_transl": np.abs(u - sl_translation(F_T, y)).max(),
         "dl_const": np.abs(v - chi * Q_C[:, None]).max()}
    blk, u, v = runs["rigid"]
    y = blk.tgt_xyz
    chi = chi_of_b(blk.tgt_b)
    e["sl_rot"] = np.abs(u - sl_rotation(OMEGA, y)).max()
    e["dl_rigid"] = np.abs(v - chi * RigidField(**RIGID)(y)).max()
    blk, u, v = runs["shear"]
    y = blk.tgt_xyz
    chi = chi_of_b(blk.tgt_b)
    e["green"] = np.abs(u + v - chi * (SHEAR_VELOCITY @ y)).max()
    return e


def test_sphere_closed_forms_and_h5_convergence(sphere_runs):
    """SL translation / rotation, DL rigid motion, DL constant (exact), Green's
    identity on the unit sphere; errors at 1/h = 32 small and falling by > 2^3.5
    from 1/h = 16 (about O(h^5) for rho = (2,3,4))."""
    e16 = _errors(sphere_runs[16])
    e32 = _errors(sphere_runs[32])
    assert e16["dl_const"] < 1e-14 and e32["dl_const"] < 1e-14  # every pair term vanishes
    limits32 = {"sl_transl": 2e-6, "sl_rot": 2e-6, "dl_rigid": 2e-5, "green": 3e-5}
    for k, lim in limits32.items():
        assert e32[k] < lim, (k, e32[k])
        assert e16[k] / e32[k] > 2 ** 3.5, (k, e16[k], e32[k])


def test_regularization_without_extrapolation_is_first_order(oracle_mod):
    """The single-delta error is O(delta): u^d1 misses the closed
    form by far more than the extrapolated u does -- pins that the solve is used."""
    blk = config1(f_field=ConstField(F_T), q_field=ZeroField(), inv_h=16, per_class=8)
    ud, _ = oracle_mod.eval_deltas_block(blk, mode=1, localized=True)
    u, _ = oracle_mod.evaluate_block(blk, mode=1, localized=True)
    ex = sl_translation(F_T, blk.tgt_xyz)
    assert np.abs(ud[0] - ex).max() > 1e-3
    assert np.abs(u - ex).max() < 2e-5


def test_localized_equals_definition(oracle_mod):
    """sharing the unregularized far part changes the totals by
    at most the s-factor deficit at t = 6 (<= 4e-14 per pair)."""
    blk = config2(inv_h=16)
    blk = blk.take_targets(np.arange(0, blk.M, 13))
    ud, vd = oracle_mod.eval_deltas_block(blk, localized=False)
    ul, vl = oracle_mod.eval_deltas_block(blk, localized=True)
    for a, b in ((ud, ul), (vd, vl)):
        assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()


@pytest.mark.parametrize("r_over_h", [11.0, 12.03, 17.5, 18.02, 23.9])
def test_near_pairs_use_exact_s_factors(oracle_mod, r_over_h):
    """Reading R1 (SURVEY 8(c) reading 1): near iff r <= 6 delta_max, and a near
    pair evaluates the exact s-factors for EVERY delta, also for the delta_k it
    lies beyond 6 delta_k of.  rho = (2, 3, 4): r = 12.03 h is beyond 6 delta_1 only,
    18.02 h beyond 6 delta_1 and 6 delta_2.  Pair by pair against 50-digit mpmath;
    just past the cutoffs a per-delta rule (s = 1 beyond 6 delta_k, the other
    reading of PAPER.md:175) differs by ~4e-14, far above this pin's tolerance."""
    blk = one_pair_block(r_over_h)
    ref = hp.brute_deltas(blk, [0])
    ud, vd = oracle_mod.eval_deltas_block(blk, localized=True)
    for k in range(3):
        ur = np.array([float(ref[k][0][i][0]) for i in range(3)])
        vr = np.array([float(ref[k][1][i][0]) for i in range(3)])
        np.testing.assert_allclose(ud[k][:, 0], ur, rtol=0, atol=2e-15 * np.abs(ur).max())
        np.testing.assert_allclose(vd[k][:, 0], vr, rtol=0, atol=2e-15 * np.abs(vr).max())
    if 12.0 < r_over_h < 12.1:  # the two readings are distinguishable here
        rule = hp.brute_deltas(blk, [0], cutoff=6)
        v_rule = np.array([float(rule[0][1][i][0]) for i in range(3)])
        v_exact = np.array([float(ref[0][1][i][0]) for i in range(3)])
        assert np.abs(v_exact - v_rule).max() > 1e-14 * np.abs(v_exact).max()


def test_brute_force_mpmath_tiny(oracle_mod):
    """Definition mode vs a 50-digit brute force on a tiny sphere (1/h = 4,
    N = 56+), 7 targets (one per b-class), cubic densities."""
    blk = config1(inv_h=4, per_class=1)
    targets = list(range(blk.M))
    ref = hp.brute_deltas(blk, targets)
    ud, vd = oracle_mod.eval_deltas_block(blk, localized=False)
    for k in range(3):
        ur = np.array([[float(x) for x in row] for row in ref[k][0]])
        vr = np.array([[float(x) for x in row] for row in ref[k][1]])
        assert np.abs(ud[k] - ur).max() <= 1e-14 * np.abs(ur).max()
        assert np.abs(vd[k] - vr).max() <= 1e-14 * np.abs(vr).max()


def test_brute_force_self_pair_limit(oracle_mod):
    """An on-surface target coinciding with a node (r = 0, reading R3) against the
    mpmath brute force with the analytic limits."""
    from workloads.configs import make_block
    from workloads.densities import PolyField
    from workloads.quadrature import quadrature, sphere
    h = 1 / 4
    x, n, w, _ = quadrature(sphere(), h)
    rng = np.random.default_rng(11)
    pick = np.array([0, 5, 17])
    blk = make_block(sphere(), h, x[:, pick], np.zeros(3), x[:, pick], n[:, pick], PolyField(rng), PolyField(rng),
                     src=(x, n, w))
    ref = hp.brute_deltas(blk, [0, 1, 2])
    ud, vd = oracle_mod.eval_deltas_block(blk, localized=False)
    for k in range(3):
        ur = np.array([[float(v) for v in row] for row in ref[k][0]])
        vr = np.array([[float(v) for v in row] for row in ref[k][1]])
        assert np.abs(ud[k] - ur).max() <= 1e-14 * np.abs(ur).max()
        assert np.abs(vd[k] - vr).max() <= 1e-14 * np.abs(vr).max()


def test_linearity_and_mode_split(oracle_mod):
    """SL is linear in f, DL in q; mode BOTH = SL run + DL run."""
    blk = config1(inv_h=16, per_class=4)
    u, v = oracle_mod.evaluate_block(blk)
    u1, _ = oracle_mod.evaluate_block(blk, mode=1)
    _, v2 = oracle_mod.evaluate_block(blk, mode=2)
    np.testing.assert_array_equal(u, u1)
    np.testing.assert_array_equal(v, v2)
    import dataclasses
    blk2 = dataclasses.replace(blk, f=2.5 * blk.f, tgt_x0_density=blk.tgt_x0_density.copy())
    blk2.tgt_x0_density[3:6] *= 2.5
    u2, _ = oracle_mod.evaluate_block(blk2, mode=1)
    np.testing.assert_allclose(u2, 2.5 * u, rtol=1e-13, atol=1e-14)


def test_invalid_arguments(oracle_mod):
    blk = config1(inv_h=8, per_class=1)
    with pytest.raises(ValueError):
        oracle_mod.evaluate(*blk.arrays(), -1.0, blk.rho)
    with pytest.raises(ValueError):
        oracle_mod.evaluate(*blk.arrays(), blk.h, (3.0, 3.0, 4.0))


# ------------------------------------------------- NEXT-1: on-surface s# variant
def _surface_block(inv_h, f_field, q_field, k=60, seed=0):
    from workloads.configs import make_block
    from workloads.quadrature import quadrature, sphere
    h = 1.0 / inv_h
    x, n, w, _ = quadrature(sphere(), h)
    pick = np.random.default_rng(seed).choice(x.shape[1], k, replace=False)
    return make_block(sphere(), h, x[:, pick], np.zeros(k), x[:, pick], n[:, pick], f_field, q_field, src=(x, n, w))


def test_sharp_on_surface_closed_forms_converge(oracle_mod):
    """s# gives O(delta^5) on the surface without extrapolation
    (delta = 3h).  SL translation/rotation and Green's identity
    (shear flow, chi = 1/2) against closed forms; error ratio 1/16 -> 1/32 > 2^4."""
    errs = {}
    for inv in (16, 32):
        h = 1.0 / inv
        e = {}
        blk = _surface_block(inv, ConstField(F_T), ConstField(Q_C))
        u, v = oracle_mod.evaluate_sharp(*blk.arrays(), 3 * h, localized=True, cutoff=7.0)
        e["sl_transl"] = np.abs(u - sl_translation(F_T, blk.tgt_xyz)).max()
        assert np.abs(v - 0.5 * Q_C[:, None]).max() < 1e-14
        blk = _surface_block(inv, RigidField(Omega=OMEGA), RigidField(**RIGID))
        u, v = oracle_mod.evaluate_sharp(*blk.arrays(), 3 * h, localized=True, cutoff=7.0)
        e["sl_rot"] = np.abs(u - sl_rotation(OMEGA, blk.tgt_xyz)).max()
        blk = _surface_block(inv, LinearField(SHEAR_TRACTION), LinearField(SHEAR_VELOCITY))
        u, v = oracle_mod.evaluate_sharp(*blk.arrays(), 3 * h, localized=True, cutoff=7.0)
        e["green"] = np.abs(u + v - 0.5 * (SHEAR_VELOCITY @ blk.tgt_xyz)).max()
        errs[inv] = e
    for k in errs[16]:
        assert errs[32][k] < 5e-7, (k, errs[32][k])
        assert errs[16][k] / errs[32][k] > 16, (k, errs[16][k], errs[32][k])


def test_sharp_brute_force_mpmath(oracle_mod):
    """oracle_eval_sharp (definition mode, no cutoff) vs the 50-digit brute force,
    including coincident-node targets (r = 0 limits of s#/t^p)."""
    from workloads.densities import PolyField
    rng = np.random.default_rng(21)
    blk = _surface_block(4, PolyField(rng), PolyField(rng), k=4, seed=3)
    delta = 3 * blk.h
    U, V = hp.brute_sharp(blk, list(range(blk.M)), delta)
    u, v = oracle_mod.evaluate_sharp(*blk.arrays(), delta, localized=False, cutoff=7.0)
    ur = np.array([[float(a) for a in row] for row in U])
    vr = np.array([[float(a) for a in row] for row in V])
    assert np.abs(u - ur).max() <= 1e-14 * np.abs(ur).max()
    assert np.abs(v - vr).max() <= 1e-14 * np.abs(vr).max()


def test_sharp_cutoff_seven(oracle_mod):
    """Reading R15: 1 - s2#(6) = 2.45e-12 is not negligible, 1 - s_i#(7) < 1e-16."""
    assert abs(1 - float(hp.s_sharp(6.0)[1])) == pytest.approx(2.45e-12, rel=0.01)
    for v in hp.s_sharp(7.0):
        assert abs(1 - float(v)) < 1e-16


def test_delta_power_schedule_next4(oracle_mod):
    """NEXT-4: delta proportional to h^q, q < 1, so that delta/h grows as
    h -> 0.  The API's h enters only through delta_k = rho_k h (the quadrature
    weights are inputs), so the schedule is the call with h_eff = C h^q:
    (i) eval(h_eff, rho) equals eval(h, rho h_eff/h) to rounding, and (ii) with
    q = 0.8 the SL-translation error still falls at high order (>= 2^3 per halving
    of h; measured 2^6.4 at these resolutions, where the discretization error, which
    the growing delta/h suppresses, still dominates the O(delta^5) regularization
    error) and at 1/h = 32 it is below the q = 1 error (the reason for q < 1)."""
    q = 0.8
    blk = config1(f_field=ConstField(F_T), q_field=ZeroField(), inv_h=16, per_class=8)
    h_eff = blk.h ** q * (1.0 / 16) ** (1 - q)
    u1, _ = oracle_mod.evaluate(*blk.arrays(), h_eff, blk.rho, mode=1, localized=True)
    u2, _ = oracle_mod.evaluate(*blk.arrays(), blk.h, tuple(r * h_eff / blk.h for r in blk.rho), mode=1,
                                localized=True)
    assert np.abs(u1 - u2).max() <= 1e-15 * np.abs(u1).max() * 10
    errs = []
    for inv in (16, 32):
        b = config1(f_field=ConstField(F_T), q_field=ZeroField(), inv_h=inv, per_class=8)
        he = b.h ** q * (1.0 / 16) ** (1 - q)
        u, _ = oracle_mod.evaluate(*b.arrays(), he, b.rho, mode=1, localized=True)
        errs.append(np.abs(u - sl_translation(F_T, b.tgt_xyz)).max())
    assert errs[0] / errs[1] > 2 ** 3, errs
    b = config1(f_field=ConstField(F_T), q_field=ZeroField(), inv_h=32, per_class=8)
    u, _ = oracle_mod.evaluate(*b.arrays(), b.h, b.rho, mode=1, localized=True)
    assert errs[1] < np.abs(u - sl_translation(F_T, b.tgt_xyz)).max()

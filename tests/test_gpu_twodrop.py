"""NEXT-2 GPU parity (-m gpu): the two-drop IE (35) pieces through the C ABI
(stokes_er_twodrop_*) against the CPU oracle (oracle/twodrop.py).

  * rhs and A u on a seeded vector: max-norm relative <= 1e-12 (north_star's
    evaluation tolerance: every piece is a sum of hot-path block evaluations)
  * the constant-density identity A c = 2 c and the lambda = 1 reduction
  * the GMRES solve: same iteration count as the oracle, residual <= 1e-10, and
    the solutions agree to 1e-8 relative (both stop at relative residual 1e-10
    of a well-conditioned second-kind system; the iterates differ by rounding)
"""
from __future__ import annotations

import numpy as np
import pytest

from workloads.twodrop import stack, twodrop

pytestmark = pytest.mark.gpu


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


@pytest.fixture(scope="module", params=[8, 16])
def case(request, ser):
    from oracle.twodrop import TwoDropOracle

    td = twodrop(request.param)
    return td, TwoDropOracle(td), ser.twodrop_solver(td)


def test_rhs_parity(case):
    td, o, s = case
    assert rel(s.rhs().cpu().numpy(), o.rhs()) <= 1e-12


def test_apply_parity(case):
    import torch

    td, o, s = case
    u = np.random.default_rng(7).uniform(-1, 1, td.n_unknowns)
    got = s.apply(torch.from_numpy(u).cuda()).cpu().numpy()
    assert rel(got, o.apply(u)) <= 1e-12


def test_constant_identity_gpu(case):
    import torch

    td, _, s = case
    c = stack([np.tile(np.array([[1.0], [-2.0], [0.5]]), (1, d.N)) for d in td.drops])
    got = s.apply(torch.from_numpy(c).cuda()).cpu().numpy()
    assert np.abs(got - 2.0 * c).max() <= 1e-13


def test_solve_parity(case):
    td, o, s = case
    u, it, hist = s.solve()
    uo, ito, histo = o.solve()
    assert it == ito and hist[-1] <= td.tol
    assert rel(u.cpu().numpy(), uo) <= 1e-8
    np.testing.assert_allclose(hist, histo, rtol=1e-6)


def test_matched_viscosity_one_step(ser):
    td = twodrop(8, lam=(1.0, 1.0))
    s = ser.twodrop_solver(td)
    u, it, hist = s.solve()
    assert it == 1
    rhs = s.rhs().cpu().numpy()
    np.testing.assert_allclose(u.cpu().numpy(), rhs / 2.0, rtol=0, atol=1e-15 * np.abs(rhs).max())


def test_setup_rejects_bad_inputs(ser):
    import torch

    td = twodrop(8)
    with pytest.raises(ser._lib.StokesERError):
        # a radius this small leaves fewer than 15 nodes in every stencil: h scaled down 8x
        bad = ser.twodrop_solver(td)
        ser.TwoDropSolver(bad._keep[0], bad._keep[1], td.h / 8, td.rho, td.delta_self)
    with pytest.raises(TypeError):
        d = [dict(x) for x in s_drops(ser, td)]
        d[0]["xyz"] = d[0]["xyz"].float()
        ser.TwoDropSolver(d, s_cross(ser, td), td.h, td.rho, td.delta_self)
    _ = torch


def s_drops(ser, td):
    return ser.twodrop_solver(td)._keep[0]


def s_cross(ser, td):
    return ser.twodrop_solver(td)._keep[1]


def test_self_convergence_matches_oracle_golden(ser):
    """GPU solves at 1/h = 8, 16: the self-convergence errors of eq. (36) equal the
    oracle's (tests/golden/twodrop_oracle.json) to 1e-6 relative."""
    import json
    import os

    from workloads.twodrop import match_nodes, split

    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "twodrop_oracle.json")))
    sols = {}
    for ih in (8, 16):
        td = twodrop(ih)
        u, it, _ = ser.twodrop_solver(td).solve()
        assert it == g["iterations"][str(ih)]
        sols[ih] = (td, u.cpu().numpy())
    idx = match_nodes(sols[8][0], sols[16][0])
    c, f = split(*sols[8]), split(*sols[16])
    e = np.concatenate([c[k] - f[k][:, idx[k]] for k in range(2)], axis=1)
    mag = np.linalg.norm(e, axis=0)
    assert abs(mag.max() / g["max_err"]["8"] - 1.0) <= 1e-6
    assert abs(np.sqrt((mag ** 2).mean()) / g["l2_err"]["8"] - 1.0) <= 1e-6


def test_twodrop_with_treecode_parity(ser):
    """NEXT-2 + NEXT-3 (the treecode on all the integrals): every block
    through the treecode on both sides (N0 300, p 8, theta 0.6) at 1/h = 16: rhs and
    A u to 1e-12, the solve to 1e-8 with the same iteration count."""
    import torch

    from oracle.twodrop import TwoDropOracle

    td = twodrop(16)
    tree = (300, 8, 0.6)
    o = TwoDropOracle(td, tree=tree)
    s = ser.twodrop_solver(td, tree=tree)
    assert rel(s.rhs().cpu().numpy(), o.rhs()) <= 1e-12
    u = np.random.default_rng(3).uniform(-1, 1, td.n_unknowns)
    assert rel(s.apply(torch.from_numpy(u).cuda()).cpu().numpy(), o.apply(u)) <= 1e-12
    ug, it, _ = s.solve()
    uo, ito, _ = o.solve()
    assert it == ito and rel(ug.cpu().numpy(), uo) <= 1e-8


def test_solve_reports_no_convergence(ser):
    """max_iter below the iterations needed: ENOCONV (include/stokes_er.h), not a silent result."""
    s = ser.twodrop_solver(twodrop(8), max_iter=3)
    with pytest.raises(ser._lib.StokesERError) as e:
        s.solve()
    assert e.value.status == 5


def test_unequal_drop_sizes(ser):
    """N1 != N2 (drop 2 thinned: not a good quadrature, but the same inputs on both sides):
    rhs and A u against the oracle."""
    import torch

    from oracle.twodrop import TwoDropOracle
    from workloads.twodrop import Cross, Drop, TwoDrop

    td = twodrop(8)
    d2 = td.drops[1]
    keep = np.arange(d2.N) % 5 != 0
    nd2 = Drop(d2.center, np.ascontiguousarray(d2.x[:, keep]), np.ascontiguousarray(d2.n[:, keep]),
               np.ascontiguousarray(d2.w[keep]), np.ascontiguousarray(d2.f[:, keep]), d2.lam)
    c1 = td.cross[1]
    nc1 = Cross(1, 0, np.ascontiguousarray(c1.b[keep]), np.ascontiguousarray(c1.x0[:, keep]),
                np.ascontiguousarray(c1.n0[:, keep]), np.ascontiguousarray(c1.f0[:, keep]))
    t2 = TwoDrop(td.h, [td.drops[0], nd2], [td.cross[0], nc1], td.rho, td.delta_self, td.tol, dict(td.meta))
    assert t2.drops[0].N != t2.drops[1].N
    o = TwoDropOracle(t2)
    s = ser.twodrop_solver(t2)
    assert rel(s.rhs().cpu().numpy(), o.rhs()) <= 1e-12
    u = np.random.default_rng(5).uniform(-1, 1, t2.n_unknowns)
    assert rel(s.apply(torch.from_numpy(u).cuda()).cpu().numpy(), o.apply(u)) <= 1e-12

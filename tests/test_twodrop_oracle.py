"""NEXT-2 pins (CPU, -m "not gpu"): the two-drop inputs and the oracle of IE (35)
(Sec. 4.3) against what the paper and the mathematics fix.

  * [f] = 2 gamma H n - grad_S gamma at points where it is known by hand
  * the interpolation (R20) reproduces degree-4 tangent polynomials
    exactly and converges at high order on a smooth function
  * lambda = 1: the DL terms vanish, A = 2 I, GMRES returns rhs/2 in one step
  * constant density: every subtracted DL pair term is 0, so A c = 2 c exactly
  * rigid motion on one drop: A q = 2 q up to the discretization error
  * the solve: GMRES residuals non-increasing, iteration count h-independent and
    within Table 2's 12-13, self-convergence max error of the
    right size and order (Table 2: 3.17e-3 at h = 1/16 against 1/32)
"""
from __future__ import annotations

import json
import os

import numpy as np
import pytest

from workloads.twodrop import EPS_PAPER, jump_force, match_nodes, split, stack, twodrop

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


@pytest.fixture(scope="module")
def td8():
    return twodrop(8)


@pytest.fixture(scope="module")
def or8(td8):
    from oracle.twodrop import TwoDropOracle

    return TwoDropOracle(td8)


def test_jump_force_by_hand():
    """[f] on the unit sphere at the origin, gamma = 1 + x1^2:
    at (0,0,1): gamma = 1, grad gamma = 0 -> 2n = (0,0,2); at (1,0,0): gamma = 2,
    grad gamma = (2,0,0) is normal, so grad_S gamma = 0 -> 4n; at (0,1,0): (0,2,0);
    at (s,s,0)/|.|, s = 1/sqrt2: gamma = 1.5, grad = (sqrt2,0,0),
    grad_S = grad - (n.grad) n = (sqrt2/2, -sqrt2/2, 0)."""
    s = 1.0 / np.sqrt(2.0)
    x = np.array([[0.0, 1.0, 0.0, s], [0.0, 0.0, 1.0, s], [1.0, 0.0, 0.0, 0.0]])
    f = jump_force(x, np.zeros(3))
    np.testing.assert_allclose(f[:, 0], [0, 0, 2], atol=1e-15)
    np.testing.assert_allclose(f[:, 1], [4, 0, 0], atol=1e-15)
    np.testing.assert_allclose(f[:, 2], [0, 2, 0], atol=1e-15)
    np.testing.assert_allclose(f[:, 3], 3.0 * np.array([s, s, 0]) - np.array([s, -s, 0]), atol=1e-15)
    # second drop: gamma uses x_c = 2 (its centre)
    c2 = np.array([2.0, 0.0, EPS_PAPER])
    f2 = jump_force(c2[:, None] + np.array([[-1.0], [0.0], [0.0]]), c2)
    np.testing.assert_allclose(f2[:, 0], [-4, 0, 0], atol=1e-15)


def test_twodrop_geometry(td8):
    """Centres (0,0,0) and (2 + 1/16^3, 0, 0) (R17); every node
    of one drop is outside the other (b' > 0) and y = x0 + b' n0 with x0 on the other
    sphere; the literal (2, 0, 1/16^3) is separation "z"."""
    for b in range(2):
        cr = td8.cross[b]
        assert cr.b.min() > 0.0
        m = td8.drops[cr.src]
        np.testing.assert_allclose(np.linalg.norm(cr.x0 - m.center[:, None], axis=0), 1.0, atol=1e-14)
        np.testing.assert_allclose(cr.x0 + cr.b * cr.n0, td8.drops[b].x, atol=1e-14)
    np.testing.assert_array_equal(td8.drops[1].center, [2.0 + EPS_PAPER, 0.0, 0.0])
    assert min(c.b.min() for c in td8.cross) >= EPS_PAPER - 1e-15
    lit = twodrop(8, separation="z")
    np.testing.assert_array_equal(lit.drops[1].center, [2.0, 0.0, EPS_PAPER])
    assert min(c.b.min() for c in lit.cross) >= np.sqrt(4.0 + EPS_PAPER ** 2) - 2.0 - 1e-15


def test_interp_reproduces_tangent_polynomials(td8):
    """Degree <= 4 polynomials in the tangent coordinates are fitted exactly (LSQ of a
    consistent system), so the stencil returns P(0, 0)."""
    from oracle.twodrop import INTERP_RADIUS, interp_weights, monomials, tangent_frame

    d = td8.drops[1]
    cr = td8.cross[0]
    rng = np.random.default_rng(3)
    pick = rng.choice(cr.b.size, 12, replace=False)
    st = interp_weights(d.x, cr.x0[:, pick], cr.n0[:, pick], td8.h)
    R = INTERP_RADIUS * td8.h
    for j, (idx, L) in zip(pick, st):
        c = rng.uniform(-1, 1, 15)
        t1, t2 = tangent_frame(cr.n0[:, j])
        rel = d.x[:, idx] - cr.x0[:, j:j + 1]
        vals = monomials(t1 @ rel / R, t2 @ rel / R) @ c
        assert abs(vals @ L - c[0]) <= 1e-12
        assert abs(L.sum() - 1.0) <= 1e-13  # constants: the weights sum to 1


def test_interp_converges_high_order():
    """u = sin(x1) + x2^2 x3 + exp(x3) on drop 2, interpolated at drop 1's closest
    points: max error falls >= 2^4 per halving of h (degree-4 fit: O(h^5))."""
    from oracle.twodrop import interp_weights

    errs = []
    for ih in (8, 16):
        td = twodrop(ih)
        d = td.drops[1]
        cr = td.cross[0]
        near = np.nonzero(cr.b < 0.5)[0]
        fn = lambda x: np.sin(x[0]) + x[1] ** 2 * x[2] + np.exp(x[2])
        st = interp_weights(d.x, cr.x0[:, near], cr.n0[:, near], td.h)
        got = np.array([fn(d.x[:, idx]) @ L for idx, L in st])
        errs.append(np.abs(got - fn(cr.x0[:, near])).max())
    assert errs[0] < 1e-4
    assert errs[0] / errs[1] > 16.0, errs


def test_matched_viscosity_reduces_to_2I():
    """lambda_1 = lambda_2 = 1: (lambda - 1) = 0 kills both DL terms, A u = 2u
    exactly, and GMRES returns rhs/2 after one step."""
    from oracle.twodrop import TwoDropOracle

    td = twodrop(8, lam=(1.0, 1.0))
    o = TwoDropOracle(td)
    u = np.random.default_rng(1).uniform(-1, 1, td.n_unknowns)
    np.testing.assert_array_equal(o.apply(u), 2.0 * u)
    sol, it, hist = o.solve()
    assert it == 1 and hist[-1] <= 1e-14
    np.testing.assert_allclose(sol, o.rhs() / 2.0, rtol=0, atol=1e-15 * np.abs(sol).max())


def test_constant_density_identity(td8, or8):
    """u = c on both drops: self DL = chi c = c/2 exactly (every subtracted pair
    term is 0), cross DL = 0 exactly (the stencil weights sum to 1), so
    A c = (lambda + 1) c - 2 (lambda - 1) c/2 = 2c."""
    c = stack([np.tile(np.array([[1.0], [-2.0], [0.5]]), (1, d.N)) for d in td8.drops])
    np.testing.assert_allclose(or8.apply(c), 2.0 * c, rtol=0, atol=1e-13)


def test_rigid_motion_on_one_drop():
    """q = U + Omega x (x - c_1) on drop 1 and 0 on drop 2: the continuous DL of a
    rigid motion is chi q (1/2 q on the drop, 0 outside it), so A q = 2 q on drop 1
    and 0 on drop 2, up to the discretization error, which falls with h."""
    from oracle.twodrop import TwoDropOracle

    errs = []
    for ih in (8, 16):
        td = twodrop(ih)
        o = TwoDropOracle(td)
        d = td.drops[0]
        U = np.array([0.3, -0.2, 0.5])
        Om = np.array([0.1, 0.4, -0.3])
        q1 = U[:, None] + np.cross(Om, (d.x - d.center[:, None]).T).T
        q = stack([q1, np.zeros((3, td.drops[1].N))])
        errs.append(np.abs(o.apply(q) - 2.0 * q).max())
    assert errs[0] < 3e-2 and errs[1] < errs[0] / 16.0, errs  # ~h^5 (measured 1.3e-2 -> 4.1e-4)


def test_gmres_solve_h8(td8, or8):
    """GMRES on IE (35) at h = 1/8: residuals non-increasing, converged to 1e-10
     in 10-15 iterations (Table 2: 13 at 1/16, 12 after,
    PAPER.md:357-365), and the solution satisfies A u = rhs."""
    u, it, hist = or8.solve()
    assert 10 <= it <= 15 and hist[-1] <= 1e-10
    assert all(b <= a * (1 + 1e-12) for a, b in zip(hist, hist[1:]))
    rhs = or8.rhs()
    assert np.linalg.norm(or8.apply(u) - rhs) <= 2e-10 * np.linalg.norm(rhs)


def test_self_convergence_golden():
    """Self-convergence e_h = u_h - u_{h/2} at the coarse nodes (eq. (36)), from
    tests/golden/twodrop_oracle.json (written by tools/gen_twodrop_golden.py,
    which calls only oracle/): the max error at 1/h = 16 is of the size Table 2
    prints (3.17e-3) and the observed order is high (Table 2: 4.89
    from 1/16 to 1/32)."""
    path = os.path.join(GOLDEN, "twodrop_oracle.json")
    if not os.path.exists(path):
        pytest.skip("golden not generated")
    g = json.load(open(path))
    e = {int(k): v for k, v in g["max_err"].items()}
    l2 = {int(k): v for k, v in g["l2_err"].items()}
    # Table 2 prints 3.17e-3 / 1.19e-4 at 1/h = 16 from a treecode run with an
    # unstated interpolation (R20); the direct-sum oracle must land within a factor
    # 1.5 (max) and 2 (L2) of them -- measured 1.28x and 1.79x
    assert 3.17e-3 / 1.5 <= e[16] <= 3.17e-3 * 1.5
    assert 1.19e-4 / 2.0 <= l2[16] <= 1.19e-4 * 2.0
    assert l2[8] / l2[16] > 2.0 ** 3.5           # high order in L2 (the max sits at the contact node)
    paper_iters = {16: 13, 32: 12}               # Table 2's GMRES iteration counts (tol 1e-10)
    for k, it in g["iterations"].items():
        if int(k) in paper_iters:
            assert abs(it - paper_iters[int(k)]) <= 1, (k, it)


def test_match_nodes_nested():
    """Grid nesting (eq. (36)): every 1/8 node is a 1/16 node."""
    idx = match_nodes(twodrop(8), twodrop(16))
    assert all(len(np.unique(i)) == len(i) for i in idx)
    td = twodrop(8)
    assert [len(i) for i in idx] == [d.N for d in td.drops]
    u = np.arange(td.n_unknowns, dtype=float)
    assert np.array_equal(stack(split(td, u)), u)

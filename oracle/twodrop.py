"""CPU oracle of the two-drop interfacial Stokes flow (NEXT-2, Sec. 4.3).

TEST INFRASTRUCTURE ONLY (same rule as oracle/__init__.py): only tests/, the
smoke entry and bench.py's reference leg may call it.  It shares no code with
the CUDA path; the layer potentials come from this package's C oracle
(stokes_er_oracle.c), everything else is plain numpy written out step by step.

The integral equation (35), for x0 on drop b (mu_0 = 1):

  (lambda_b + 1) u(x0) = -(1/4pi) sum_m int_m S [f] dS + sum_m (lambda_m - 1)/(4pi) int_m T u n dS

With the evaluators' 1/(8pi) (eqs. (10)-(11)) this is, per drop b and m != b,

  A u|_b = (lambda_b + 1) u_b - 2 (lambda_b - 1) DL_bb[u_b] - 2 (lambda_m - 1) DL_bm[u_m]
  rhs_b  = -2 (SL_bb[[f]_b] + SL_bm[[f]_m])

where the self blocks (targets on the source surface) use the on-surface s#
regularization with delta = 3h (NEXT-1; DL_bb is the principal
value: chi = 1/2) and the cross blocks use the 3-delta extrapolated method with
delta = {3h, 4h, 5h}.  The cross DL's subtraction needs u_m at
the closest point x0 on drop m, which is not a node: DESIGN.md R20 reads it as
a degree-4 least-squares fit in the tangent plane of x0 over the nodes within
3.5h (`interp_weights`), at every cross target.  GMRES:
full, modified Gram-Schmidt, x_0 = 0, stop at ||b - A u|| <= 1e-10 ||b||
(R21).
"""
from __future__ import annotations

import numpy as np

from . import BOTH, DL, SL, evaluate, evaluate_sharp, evaluate_tree, evaluate_tree_sharp

INTERP_RADIUS = 3.5      # neighbours within 3.5 h of x0 (R20)
INTERP_DEGREE = 4        # total degree in the tangent coordinates: 15 monomials
CUTOFF = 6.0             # extrapolated blocks: near iff r <= 6 delta_max (R1)
CUTOFF_SHARP = 7.0       # s# blocks (R15)


def monomials(xi, eta, degree=INTERP_DEGREE):
    """Columns xi^a eta^b, a + b <= degree, constant first."""
    cols = [xi ** (d - b) * eta ** b for d in range(degree + 1) for b in range(d + 1)]
    return np.stack(cols, axis=1)


def tangent_frame(n0):
    """Any orthonormal t1, t2 with n0 (the fitted polynomial space is rotation invariant)."""
    e = np.zeros(3)
    e[int(np.argmin(np.abs(n0)))] = 1.0
    t1 = np.cross(n0, e)
    t1 /= np.linalg.norm(t1)
    return t1, np.cross(n0, t1)


def interp_weights(nodes, x0, n0, h, radius=INTERP_RADIUS, degree=INTERP_DEGREE):
    """Least-squares interpolation at x0 on the node surface (R20).

    For each point x0[:, t]: neighbours = nodes within radius*h; tangent
    coordinates (xi, eta) = ((x_k - x0).t1, (x_k - x0).t2) / (radius h); the value
    at x0 of the least-squares polynomial of total degree <= degree is
    sum_k L_k u(x_k) with L = first row of pinv(Phi).
    Returns a list of (indices, weights)."""
    from scipy.spatial import cKDTree

    tree = cKDTree(nodes.T)
    R = radius * h
    out = []
    for t in range(x0.shape[1]):
        idx = np.array(sorted(tree.query_ball_point(x0[:, t], R)), dtype=np.int64)
        t1, t2 = tangent_frame(n0[:, t])
        d = nodes[:, idx] - x0[:, t:t + 1]
        phi = monomials(t1 @ d / R, t2 @ d / R, degree)
        if idx.size < phi.shape[1]:
            raise ValueError(f"interp: only {idx.size} nodes within {radius} h")
        out.append((idx, np.linalg.pinv(phi)[0]))
    return out


class TwoDropOracle:
    """Operator, right-hand side and GMRES solve of IE (35) on the CPU."""

    def __init__(self, td, localized=True, nthreads=0, tree=None):
        """tree: None (direct localized sums) or (leaf_size, degree, theta): every block
        through the treecode oracle (NEXT-3)."""
        self.td = td
        self.tree = tree
        self.localized = localized
        self.nthreads = nthreads
        self.interp = []   # per drop b: interpolation stencils on drop 1-b at its nodes' x0
        for b in range(2):
            cr = td.cross[b]
            self.interp.append(interp_weights(td.drops[cr.src].x, cr.x0, cr.n0, td.h))

    # ---- blocks -------------------------------------------------------------------------
    def _self(self, b, f=None, q=None, mode=DL):
        d = self.td.drops[b]
        N = d.N
        x0d = np.zeros((9, N))
        x0d[0:3] = d.n
        if f is not None:
            x0d[3:6] = f
        if q is not None:
            x0d[6:9] = q
        z = np.zeros((3, N))
        args = (d.x, d.n, d.w, f if f is not None else z, q if q is not None else z, d.x, np.zeros(N), x0d,
                self.td.delta_self)
        if self.tree is not None:
            return evaluate_tree_sharp(*args, *self.tree, mode=mode, nthreads=self.nthreads)
        return evaluate_sharp(*args, mode=mode, localized=self.localized, cutoff=CUTOFF_SHARP,
                              nthreads=self.nthreads)

    def q0_cross(self, b, u_src):
        """u_{1-b} at the closest points x0 of drop b's nodes (R20)."""
        q0 = np.zeros((3, self.td.drops[b].N))
        for t, (idx, L) in enumerate(self.interp[b]):
            q0[:, t] = u_src[:, idx] @ L
        return q0

    def _cross(self, b, f=None, q=None, mode=DL):
        cr = self.td.cross[b]
        src = self.td.drops[cr.src]
        tgt = self.td.drops[b]
        x0d = np.zeros((9, tgt.N))
        x0d[0:3] = cr.n0
        x0d[3:6] = cr.f0
        if q is not None:
            x0d[6:9] = self.q0_cross(b, q)
        z = np.zeros((3, src.N))
        args = (src.x, src.n, src.w, f if f is not None else z, q if q is not None else z, tgt.x, cr.b, x0d,
                self.td.h, self.td.rho)
        if self.tree is not None:
            return evaluate_tree(*args, *self.tree, mode=mode, nthreads=self.nthreads)
        return evaluate(*args, mode=mode, localized=self.localized, nthreads=self.nthreads)

    # ---- IE (35) -----------------------------------------------------------------------
    def rhs(self):
        """-(1/(4 pi mu_0)) sum_m int S [f] = -2 (SL_bb + SL_bm), per drop, stacked."""
        parts = []
        for b in range(2):
            m = 1 - b
            u_self, _ = self._self(b, f=self.td.drops[b].f, mode=SL)
            u_cross, _ = self._cross(b, f=self.td.drops[m].f, mode=SL)
            parts.append(-2.0 * (u_self + u_cross))
        return np.concatenate([p.reshape(-1) for p in parts])

    def apply(self, vec):
        """A u (stacked (3 N_1 + 3 N_2,) vectors)."""
        n1 = self.td.drops[0].N
        u = [vec[:3 * n1].reshape(3, n1), vec[3 * n1:].reshape(3, self.td.drops[1].N)]
        parts = []
        for b in range(2):
            m = 1 - b
            lb, lm = self.td.drops[b].lam, self.td.drops[m].lam
            _, v_self = self._self(b, q=u[b], mode=DL)
            _, v_cross = self._cross(b, q=u[m], mode=DL)
            parts.append((lb + 1.0) * u[b] - 2.0 * (lb - 1.0) * v_self - 2.0 * (lm - 1.0) * v_cross)
        return np.concatenate([p.reshape(-1) for p in parts])

    def solve(self, tol=None, max_iter=100):
        """Full GMRES with modified Gram-Schmidt from u = 0 (R21).

        Returns (u stacked, iterations, residual history ||r_j|| / ||b||)."""
        tol = self.td.tol if tol is None else tol
        b = self.rhs()
        beta = np.linalg.norm(b)
        n = b.size
        V = np.zeros((max_iter + 1, n))
        H = np.zeros((max_iter + 1, max_iter))
        V[0] = b / beta
        hist = []
        y = np.zeros(0)
        for j in range(max_iter):
            w = self.apply(V[j])
            for i in range(j + 1):
                H[i, j] = w @ V[i]
                w = w - H[i, j] * V[i]
            H[j + 1, j] = np.linalg.norm(w)
            if H[j + 1, j] > 0.0:
                V[j + 1] = w / H[j + 1, j]
            e1 = np.zeros(j + 2)
            e1[0] = beta
            y = np.linalg.lstsq(H[:j + 2, :j + 1], e1, rcond=None)[0]
            res = np.linalg.norm(e1 - H[:j + 2, :j + 1] @ y) / beta
            hist.append(res)
            if res <= tol or H[j + 1, j] == 0.0:
                break
        u = V[:len(y)].T @ y
        return u, len(hist), hist

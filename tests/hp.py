"""50-digit mpmath evaluations used to pin the oracle (test-only).

Written from PAPER.md directly, in a different arrangement from the oracle
where one exists, so a transcription slip in either shows up:

* s-factors, eqs. (14)-(16) and s#
* I0, I2, eqs. (18)-(19)
* brute-force per-delta sums of eqs. (10)-(13).  The
  stresslet uses the equivalent arrangement
      T^d_iac = -6 [ s3 yh_i yh_a yh_c / r^5 + (s2 - s3) t1_iac / r^3 ]
  which follows from eq. (7) with t2 = yh yh yh - b^2 t1 (expand
  yh = b n0 - xh); the oracle uses the t1/t2 form literally.
"""
from __future__ import annotations

import mpmath as mp

mp.mp.dps = 50
SQPI = mp.sqrt(mp.pi)


def s_factors(t):
    t = mp.mpf(t)
    E = mp.erf(t)
    G = 2 / SQPI * mp.exp(-t * t)
    return E, E - G * t, E - G * (t + mp.mpf(2) / 3 * t ** 3)


def s_sharp(t):
    t = mp.mpf(t)
    E = mp.erf(t)
    e = mp.exp(-t * t)
    return (E + 2 / (3 * SQPI) * (5 * t - 2 * t ** 3) * e,
            E - 2 / (3 * SQPI) * (3 * t - 14 * t ** 3 + 4 * t ** 5) * e,
            E - 2 / (9 * SQPI) * (9 * t + 6 * t ** 3 - 4 * t ** 5) * e)


def I0(lam):
    lam = mp.mpf(lam)
    a = abs(lam)
    return mp.exp(-lam ** 2) / SQPI - a * mp.erfc(a)


def I2(lam):
    lam = mp.mpf(lam)
    a = abs(lam)
    return mp.mpf(2) / 3 * ((mp.mpf(1) / 2 - lam ** 2) * mp.exp(-lam ** 2) / SQPI + a ** 3 * mp.erfc(a))


def _reg(r, d):
    """(s1/r, s2/r^3, s3/r^5) with the exact r -> 0 limits."""
    if r == 0:
        return 2 / (SQPI * d), 4 / (3 * SQPI * d ** 3), 8 / (15 * SQPI * d ** 5)
    s1, s2, s3 = s_factors(r / d)
    return s1 / r, s2 / r ** 3, s3 / r ** 5


def brute_deltas(block, targets, mode=3, cutoff=None):
    """Definition-mode u^dk, v^dk at 50 digits for the listed target indices.
    With `cutoff`, s1 = s2 = s3 = 1 for r > cutoff * delta_k (the per-delta
    reading of PAPER.md:175 that DESIGN.md R1 does not take; pins tell the two apart).
    Returns dict k -> (u list[3][T], v list[3][T]) as mpf."""
    N = block.N
    X = [[mp.mpf(float(block.src_xyz[i, s])) for s in range(N)] for i in range(3)]
    Nn = [[mp.mpf(float(block.src_normal[i, s])) for s in range(N)] for i in range(3)]
    W = [mp.mpf(float(w)) for w in block.src_weight]
    Fd = [[mp.mpf(float(block.f[i, s])) for s in range(N)] for i in range(3)]
    Qd = [[mp.mpf(float(block.q[i, s])) for s in range(N)] for i in range(3)]
    deltas = [mp.mpf(r) * mp.mpf(block.h) for r in block.rho]
    out = {k: ([[None] * len(targets) for _ in range(3)], [[None] * len(targets) for _ in range(3)])
           for k in range(3)}
    for ti, t in enumerate(targets):
        y = [mp.mpf(float(block.tgt_xyz[i, t])) for i in range(3)]
        b = mp.mpf(float(block.tgt_b[t]))
        n0 = [mp.mpf(float(block.tgt_x0_density[i, t])) for i in range(3)]
        f0 = [mp.mpf(float(block.tgt_x0_density[3 + i, t])) for i in range(3)]
        q0 = [mp.mpf(float(block.tgt_x0_density[6 + i, t])) for i in range(3)]
        x0 = [y[i] - b * n0[i] for i in range(3)]
        alpha = sum(f0[i] * n0[i] for i in range(3))
        chi = mp.mpf(1) if b < 0 else (mp.mpf(0) if b > 0 else mp.mpf(1) / 2)
        U = [[mp.mpf(0)] * 3 for _ in range(3)]
        V = [[mp.mpf(0)] * 3 for _ in range(3)]
        for s in range(N):
            yh = [y[i] - X[i][s] for i in range(3)]
            xh = [X[i][s] - x0[i] for i in range(3)]
            m = [Nn[i][s] for i in range(3)]
            r = mp.sqrt(sum(c * c for c in yh))
            g = [Fd[a][s] - alpha * m[a] for a in range(3)]
            dq = [Qd[a][s] - q0[a] for a in range(3)]
            yg = sum(yh[a] * g[a] for a in range(3))
            yq = sum(yh[a] * dq[a] for a in range(3))
            ym = sum(yh[c] * m[c] for c in range(3))
            # t1 contracted with dq_a m_c (eq. 8)
            nq = sum(n0[a] * dq[a] for a in range(3))
            nm = sum(n0[c] * m[c] for c in range(3))
            xq = sum(xh[a] * dq[a] for a in range(3))
            xm = sum(xh[c] * m[c] for c in range(3))
            t1c = [b * n0[i] * nq * nm - (xh[i] * nq * nm + n0[i] * xq * nm + n0[i] * nq * xm) for i in range(3)]
            for k, d in enumerate(deltas):
                if cutoff is not None and r > cutoff * d:
                    A1, A3, A5 = 1 / r, 1 / r ** 3, 1 / r ** 5
                    s2ms3_r3 = mp.mpf(0)
                elif r == 0:
                    A1, A3, A5 = _reg(r, d)
                    s2ms3_r3 = 4 / (3 * SQPI * d ** 3)
                else:
                    s1, s2, s3 = s_factors(r / d)
                    A1, A3, A5 = s1 / r, s2 / r ** 3, s3 / r ** 5
                    s2ms3_r3 = (s2 - s3) / r ** 3
                for i in range(3):
                    U[k][i] += W[s] * (g[i] * A1 + yh[i] * yg * A3)
                    V[k][i] += W[s] * (-6) * (A5 * yh[i] * yq * ym + s2ms3_r3 * t1c[i])
        for k in range(3):
            for i in range(3):
                out[k][0][i][ti] = U[k][i] / (8 * mp.pi)
                out[k][1][i][ti] = V[k][i] / (8 * mp.pi) + chi * q0[i]
    return out


def brute_sharp(block, targets, delta, cutoff=None):
    """NEXT-1 on-surface variant at 50 digits: S^d with s1#, s2# (eq. 12 with the
    s# of PAPER.md:130-138) and the unsplit stresslet times s3# (R16).
    `cutoff` (in units of delta) applies s# = 1 beyond it, as the localized oracle does.
    Returns (u list[3][T], v list[3][T])."""
    N = block.N
    d = mp.mpf(delta)
    U = [[None] * len(targets) for _ in range(3)]
    V = [[None] * len(targets) for _ in range(3)]
    for ti, t in enumerate(targets):
        y = [mp.mpf(float(block.tgt_xyz[i, t])) for i in range(3)]
        b = mp.mpf(float(block.tgt_b[t]))
        n0 = [mp.mpf(float(block.tgt_x0_density[i, t])) for i in range(3)]
        f0 = [mp.mpf(float(block.tgt_x0_density[3 + i, t])) for i in range(3)]
        q0 = [mp.mpf(float(block.tgt_x0_density[6 + i, t])) for i in range(3)]
        alpha = sum(f0[i] * n0[i] for i in range(3))
        chi = mp.mpf(1) if b < 0 else (mp.mpf(0) if b > 0 else mp.mpf(1) / 2)
        u = [mp.mpf(0)] * 3
        v = [mp.mpf(0)] * 3
        for s in range(N):
            x = [mp.mpf(float(block.src_xyz[i, s])) for i in range(3)]
            m = [mp.mpf(float(block.src_normal[i, s])) for i in range(3)]
            w = mp.mpf(float(block.src_weight[s]))
            yh = [y[i] - x[i] for i in range(3)]
            r = mp.sqrt(sum(c * c for c in yh))
            g = [mp.mpf(float(block.f[a, s])) - alpha * m[a] for a in range(3)]
            dq = [mp.mpf(float(block.q[a, s])) - q0[a] for a in range(3)]
            if r == 0:
                A1, A3, A5 = (lim / d ** p for lim, p in zip(sharp_limits(), (1, 3, 5)))
            else:
                s1, s2, s3 = s_sharp(r / d) if (cutoff is None or r / d <= cutoff) else (1, 1, 1)
                A1, A3, A5 = s1 / r, s2 / r ** 3, s3 / r ** 5
            yg = sum(yh[a] * g[a] for a in range(3))
            yq = sum(yh[a] * dq[a] for a in range(3))
            ym = sum(yh[c] * m[c] for c in range(3))
            for i in range(3):
                u[i] += w * (g[i] * A1 + yh[i] * yg * A3)
                v[i] += w * (-6) * yh[i] * yq * ym * A5
        for i in range(3):
            U[i][ti] = u[i] / (8 * mp.pi)
            V[i][ti] = v[i] / (8 * mp.pi) + chi * q0[i]
    return U, V


def sharp_limits():
    """lim_{t->0} s#_i(t)/t^p for p = 1, 3, 5, evaluated numerically at t = 1e-40 with
    400 digits (independent of the series the oracle's comments derive)."""
    with mp.workdps(400):
        t = mp.mpf(10) ** -40
        sq = mp.sqrt(mp.pi)
        E = mp.erf(t)
        e = mp.exp(-t * t)
        s1 = E + 2 / (3 * sq) * (5 * t - 2 * t ** 3) * e
        s2 = E - 2 / (3 * sq) * (3 * t - 14 * t ** 3 + 4 * t ** 5) * e
        s3 = E - 2 / (9 * sq) * (9 * t + 6 * t ** 3 - 4 * t ** 5) * e
        out = (s1 / t, s2 / t ** 3, s3 / t ** 5)
    return tuple(mp.mpf(x) for x in out)

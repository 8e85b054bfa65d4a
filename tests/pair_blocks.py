"""Single-pair blocks for pair-level pins (shared by the oracle pins and the GPU parity tests)."""
from __future__ import annotations

import numpy as np


def one_pair_block(r_over_h, h=1 / 64, seed=5):
    """One source at the origin, one target at distance r_over_h * h along a
    random direction, random densities (a pair-level pin)."""
    from workloads.configs import Block
    rng = np.random.default_rng(seed)
    m = rng.standard_normal(3); m /= np.linalg.norm(m)
    e = rng.standard_normal(3); e /= np.linalg.norm(e)
    y = e * r_over_h * h
    n0 = rng.standard_normal(3); n0 /= np.linalg.norm(n0)
    b = 0.3 * h
    col = lambda v: np.ascontiguousarray(np.asarray(v, float).reshape(-1, 1))
    x0d = np.concatenate([n0, rng.standard_normal(3), rng.standard_normal(3)])
    return Block(src_xyz=col(np.zeros(3)), src_normal=col(m), src_weight=np.array([0.7]),
                 f=col(rng.standard_normal(3)), q=col(rng.standard_normal(3)), tgt_xyz=col(y),
                 tgt_b=np.array([b]), tgt_x0_density=col(x0d), h=h, rho=(2.0, 3.0, 4.0))

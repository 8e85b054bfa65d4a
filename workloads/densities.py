"""Seeded input generation, part 2: density fields f, q evaluated at nodes and at x0.

Only input fields live here (BASELINE.json configs): seeded cubic polynomials,
seeded products of sines/cosines, and the closed-form cases used by the
oracle pins (constant translation, rotation, rigid motion, Stokes shear).
No hot-path arithmetic.
"""
from __future__ import annotations

import itertools

import numpy as np

# monomial exponents alpha with |alpha| <= 3 (20 of them), fixed order
MONOMIALS_DEG3 = [a for d in range(4) for a in itertools.product(range(4), repeat=3) if sum(a) == d]
assert len(MONOMIALS_DEG3) == 20


class Field:
    """A vector field R^3 -> R^3 evaluated on (3, K) arrays."""

    def __call__(self, x):  # pragma: no cover - interface
        raise NotImplementedError


class PolyField(Field):
    """Per component sum_{|alpha|<=3} c_alpha x^alpha, c ~ U[-1,1] (configs 1, 2, 4, 5)."""

    def __init__(self, rng: np.random.Generator):
        self.coef = rng.uniform(-1.0, 1.0, size=(3, len(MONOMIALS_DEG3)))

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        mono = np.stack([x[0] ** a[0] * x[1] ** a[1] * x[2] ** a[2] for a in MONOMIALS_DEG3])
        return self.coef @ mono


class TrigField(Field):
    """f_j = sum_{m=1..4} a_jm prod_l tau_jml(kappa_jml x_l + phi_jml) (config 3)."""

    def __init__(self, rng: np.random.Generator, terms: int = 4):
        self.a = rng.uniform(-1.0, 1.0, size=(3, terms))
        self.tau = rng.integers(0, 2, size=(3, terms, 3))  # 0 -> sin, 1 -> cos
        self.kappa = rng.integers(1, 4, size=(3, terms, 3)).astype(np.float64)
        self.phi = rng.uniform(0.0, 2.0 * np.pi, size=(3, terms, 3))

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64)
        out = np.zeros((3, x.shape[1]))
        for j in range(3):
            for m in range(self.a.shape[1]):
                prod = np.ones(x.shape[1])
                for l in range(3):
                    arg = self.kappa[j, m, l] * x[l] + self.phi[j, m, l]
                    prod *= np.cos(arg) if self.tau[j, m, l] else np.sin(arg)
                out[j] += self.a[j, m] * prod
        return out


class ConstField(Field):
    def __init__(self, value):
        self.value = np.asarray(value, dtype=np.float64)

    def __call__(self, x):
        return np.repeat(self.value[:, None], np.asarray(x).shape[1], axis=1)


class RigidField(Field):
    """U + Omega x (x - c)."""

    def __init__(self, U=(0.0, 0.0, 0.0), Omega=(0.0, 0.0, 0.0), center=(0.0, 0.0, 0.0)):
        self.U = np.asarray(U, dtype=np.float64)
        self.Omega = np.asarray(Omega, dtype=np.float64)
        self.center = np.asarray(center, dtype=np.float64)

    def __call__(self, x):
        x = np.asarray(x, dtype=np.float64) - self.center[:, None]
        return self.U[:, None] + np.cross(self.Omega, x.T).T


class ZeroField(ConstField):
    def __init__(self):
        super().__init__((0.0, 0.0, 0.0))


class LinearField(Field):
    """A x + U (e.g. the shear flow u = (x2, 0, 0) and its traction (x2, x1, 0) on the unit sphere)."""

    def __init__(self, A, U=(0.0, 0.0, 0.0)):
        self.A = np.asarray(A, dtype=np.float64)
        self.U = np.asarray(U, dtype=np.float64)

    def __call__(self, x):
        return self.A @ np.asarray(x, dtype=np.float64) + self.U[:, None]

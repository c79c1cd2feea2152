"""The inverse-model twin case of tests/golden/make_golden_inverse.py, shared
by the oracle and GPU parity tests (the reference's inverse_twin layout on a
16x8 / 32x16 pair of nested meshes)."""

import numpy as np

BOUNDS = (0.0, 0.0, 2.0, 1.0)
COARSE = (16, 8)
FINE = (32, 16)
CONTRAST = 10.0
LAME = (1.25, 1.0)  # the reference's default Lame pair (models/base.py:124-147)
FORCES = [((1.0, 0.0), 3), ((0.0, -1.0), 4), ((-1.0, 0.0), 5)]
FIXED = 1
MEASURED = (2, 3, 4, 5)


def rules():
    eps = 1e-12
    return [(3, lambda p: (p[:, 0] < eps) & (p[:, 1] > 0.25) & (p[:, 1] < 0.75)),
            (4, lambda p: (p[:, 1] > 1.0 - eps) & (p[:, 0] > 0.75) & (p[:, 0] < 1.25)),
            (5, lambda p: (p[:, 0] > 2.0 - eps) & (p[:, 1] > 0.25) & (p[:, 1] < 0.75)),
            (1, lambda p: p[:, 1] < eps),
            (2, lambda p: np.ones(len(p), dtype=bool))]


def inclusion(p):  # true stiff disk, negative inside
    return np.hypot(p[:, 0] - 1.0, p[:, 1] - 0.5) - 0.25


def guess(p):  # offset initial guess
    return np.hypot(p[:, 0] - 0.9, p[:, 1] - 0.6) - 0.35

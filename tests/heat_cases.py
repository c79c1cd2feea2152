"""The heat-model case of tests/golden/make_golden_heat.py, shared by the oracle
and GPU parity tests (kept in step with the generator by hand: same mesh,
tags, level set and sources)."""

import numpy as np

BOUNDS = (0.0, 0.0, 1.5, 1.0)
NX, NY = 24, 16
VOLUME = 0.6
RULES = [(1, lambda p: p[:, 0] < 1e-12),
         (2, lambda p: (p[:, 1] < 1e-12) & (p[:, 0] > 0.5) & (p[:, 0] < 1.0)),
         (3, lambda p: p[:, 0] > 1.5 - 1e-12)]


def phi_fn(p):
    return -np.cos(4 * np.pi * p[:, 0] / 1.5) * np.cos(3 * np.pi * p[:, 1]) - 0.2


def src_a(p):
    return 1.0 + 0.5 * p[:, 0] * p[:, 1]


def grad_a(p):
    return np.stack([0.5 * p[:, 1], 0.5 * p[:, 0]], axis=1)


def src_b(p):
    return np.full(len(p), 2.0)

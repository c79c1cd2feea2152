"""Descent velocities from distributed shape derivatives (drop-in for reference ``velocity.py``).

``VelocitySolver(spec, space).solve(pair)`` keeps the reference's contract
(``velocity.py:85-154``): theta solves B(theta, xi) = -dJ(xi) for all xi and
the result carries B(theta, theta) and dJ(theta).  The reference factorises B
once with SuperLU; here B is the matrix-free H1 operator (mass + alpha *
vector Laplacian, plus the optional boundary-normal / frozen / zero-Dirichlet
terms) solved by the same fused Jacobi-PCG as the state, to relative
residual 1e-12 (tighter than the state's 1e-10 because it stands in for a
direct solve and must keep the descent identity |dJ + B| <= 1e-8 (1 + B) of
``driver.py:280``).

A ``DerivativePair`` may carry, besides the reference's ``s0`` / ``s1``
closures, ``vector`` terms: device vectors that already hold
int S0 . N_a + S1 : grad(N_a e_c) -- what the fused compliance kernel
produces, so that S1 never has to be materialised on the hot path.
"""

import math
from dataclasses import dataclass, field
from typing import Callable, NamedTuple, Optional

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, SolverError
from .fem import FemField, H1Operator, solve_batched, to_device

__all__ = ["BilinearSpec", "DerivativePair", "VelocityResult", "VelocitySolver", "VELOCITY_RTOL"]

VELOCITY_RTOL = 1e-12


@dataclass(frozen=True)
class BilinearSpec:
    """Weights of the velocity form (``velocity.py:32-69``)."""

    mass_weight: float = 0.0
    stiffness_weight: float = 1.0
    boundary_normal_penalty: float = 0.0
    frozen_subdomain: Optional[Callable] = None
    frozen_penalty: float = 0.0
    zero_dirichlet: bool = False

    def __post_init__(self):
        if min(self.mass_weight, self.boundary_normal_penalty, self.frozen_penalty) < 0:
            raise ConfigError("velocity form weights must be nonnegative")
        if self.stiffness_weight <= 0:
            raise ConfigError("velocity form needs stiffness_weight > 0")
        if not (self.zero_dirichlet or self.mass_weight > 0 or self.boundary_normal_penalty > 0):
            raise ConfigError(
                "velocity form is indefinite: constants are stiffness-kernel fields; "
                "enable zero_dirichlet, a mass term, or a boundary normal penalty")
        if (self.frozen_subdomain is None) != (self.frozen_penalty == 0.0):
            raise ConfigError("frozen_subdomain and a positive frozen_penalty go together")


@dataclass(frozen=True)
class DerivativePair:
    """Tensor representation (S0, S1) of a shape derivative (``velocity.py:72-82``).

    ``s0(space) -> (E, nq, d)`` and ``s1(space) -> (E, nq, d, d)`` closures as
    in the reference; ``vector`` is a tuple of (weight, device tensor (d N,))
    terms already contracted with the test functions.
    """

    s0: Optional[Callable] = None
    s1: Optional[Callable] = None
    vector: tuple = ()


class VelocityResult(NamedTuple):
    theta: FemField
    form_value: float  # B(theta, theta)
    derivative: float  # dJ(theta)


def _quad_points(mesh):
    """Quadrature points (E, nq, d) on the host (setup only; frozen predicate)."""
    p = mesh.vertices[mesh.elements]
    if mesh.dim == 2:
        bary = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])
    else:
        a, b = 0.5854101966249685, 0.1381966011250105
        bary = np.full((4, 4), b) + np.eye(4) * (a - b)
    return np.einsum("qi,tid->tqd", bary, p)


class VelocitySolver:
    """Matrix-free velocity form, reused across all solves on one mesh."""

    def __init__(self, spec: BilinearSpec, space):
        if space.value_rank != space.dim:
            raise ConfigError("velocity solves need a vector-valued space")
        self.spec = spec
        self.space = space
        frozen_q = None
        if spec.frozen_subdomain is not None:
            pts = _quad_points(space.mesh)
            inside = np.asarray(spec.frozen_subdomain(pts.reshape(-1, space.dim)), dtype=bool)
            frozen_q = inside.reshape(pts.shape[:2]).astype(np.uint8)
        self.operator = H1Operator(space, spec.mass_weight, spec.stiffness_weight,
                                   spec.boundary_normal_penalty, frozen_q, spec.frozen_penalty,
                                   spec.zero_dirichlet)
        n = space.dof_count
        self._stats = torch.zeros(4, dtype=torch.float64, device="cuda")
        self._part = torch.zeros(int(_lib.load().lsg_partials_per_rhs(space.mesh.grid)) * 4,
                                 dtype=torch.float64, device="cuda")
        self._cnt = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._zero = torch.zeros(n, dtype=torch.float64, device="cuda")
        self.last_iterations = 0

    def _derivative_vector(self, pair: DerivativePair):
        """The vector int S0 . N_a + S1 : grad(N_a e_c) (``velocity.py:129-142``)."""
        space = self.space
        vec = torch.zeros(space.dof_count, dtype=torch.float64, device="cuda")
        for w, v in pair.vector:
            vec.add_(to_device(v), alpha=float(w))
        if pair.s0 is not None or pair.s1 is not None:
            s0 = s1 = None
            if pair.s0 is not None:
                s0 = to_device(pair.s0(space))
                if not bool(torch.isfinite(s0).all()):
                    raise ConfigError("S0 tensor has non-finite quadrature values")
            if pair.s1 is not None:
                s1 = to_device(pair.s1(space))
                if not bool(torch.isfinite(s1).all()):
                    raise ConfigError("S1 tensor has non-finite quadrature values")
            tmp = torch.empty_like(vec)
            _lib.call("lsg_tensor_rhs", space.mesh.grid, _lib.ptr(s0), _lib.ptr(s1),
                      _lib.ptr(tmp), _lib.stream())
            vec.add_(tmp)
        return vec

    def _rhs(self, pair):
        """b = -vec with Dirichlet dofs zeroed; fused single kernel for two vector terms."""
        if pair.s0 is None and pair.s1 is None and 1 <= len(pair.vector) <= 2:
            terms = list(pair.vector)
            (w0, v0) = terms[0]
            v0 = to_device(v0)
            if len(terms) == 2:
                w1, v1 = terms[1]
                v1 = to_device(v1)
            else:
                w1, v1 = 0.0, self._zero
            if w0 != 1.0:
                v0 = v0 * float(w0)
            b = torch.empty_like(v0)
            _lib.call("lsg_velocity_rhs", self.operator._op(), _lib.ptr(v0), _lib.ptr(v1),
                      float(w1), _lib.ptr(b), _lib.stream())
            return b
        vec = self._derivative_vector(pair)
        b = torch.empty_like(vec)
        _lib.call("lsg_velocity_rhs", self.operator._op(), _lib.ptr(vec), _lib.ptr(self._zero),
                  0.0, _lib.ptr(b), _lib.stream())
        return b

    def solve(self, pair: DerivativePair) -> VelocityResult:
        b = self._rhs(pair)
        x, iters = solve_batched(self.operator, b, rtol=VELOCITY_RTOL, atol=0.0)
        self.last_iterations = int(iters[0])
        theta = x[0]
        # stats: theta^T B theta, b . theta (= -vec . theta on free dofs), CFL speed
        _lib.call("lsg_velocity_stats", self.operator._op(), _lib.ptr(theta), _lib.ptr(b),
                  _lib.ptr(self._stats), _lib.ptr(self._part), _lib.ptr(self._cnt), _lib.stream())
        btt, bth, speed = self._stats[:3].tolist()
        field = FemField(self.space, theta)
        field._cfl_speed = float(speed)
        return VelocityResult(field, float(btt), float(-bth))

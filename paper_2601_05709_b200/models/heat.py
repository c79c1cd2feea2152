"""Thermal compliance models (drop-in for reference ``models/heat.py``).

Same contract as ``HeatModel`` / ``HeatPlusModel`` / ``HeatTerm``
(``heat.py:37-171``): the conductor occupies the subzero set, the complement
keeps contrast 1e-3 (``:34``); J = sum_t c_t int A |grad u_t|^2 with u_t the
temperature under source f_t grounded on the term's tags; the adjoint is
-c_t u_t and is never solved (``:124-128``); S0 = sum_t c_t 2 u grad f (only
for sources with a gradient), S1 = sum_t c_t ((2 u f - A |grad u|^2) I +
2 A grad u (x) grad u) (``:140-166``).

Device path: ``pde`` builds one ``LaplaceOperator`` per distinct ground set
(terms sharing a ground are solved as one PCG batch); ``cost`` runs the fused
thermal-compliance + shape-derivative kernel (``lsg_heat_shape``) once per
iteration over all terms and caches J, the volume and the two contracted
derivative vectors that ``constraint`` and ``derivative`` reuse.  The source
samples at the quadrature points (and the load vectors) are set up once on
the host, as the reference does.
"""

from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np
import torch

from .. import _lib
from ..errors import ConfigError
from ..fem import DirichletSet, FemField, FunctionSpace, LaplaceOperator, LinearProblem, to_device
from ..velocity import BilinearSpec, DerivativePair, _quad_points
from .base import MaterialIndicator, ModelProblem

__all__ = ["HeatModel", "HeatTerm", "HeatPlusModel", "CONTRAST"]

CONTRAST = 1e-3
_BARY = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])


@dataclass(frozen=True)
class HeatTerm:
    """One source/ground pairing of a summed thermal compliance (``heat.py:37-50``)."""

    source: Callable
    fixed_tags: object
    weight: Optional[float] = None
    source_gradient: Optional[Callable] = None


class HeatModel(ModelProblem):
    """Single-term thermal compliance with a volume constraint (``heat.py:78-166``)."""

    def __init__(self, mesh, fixed_tags, source, volume, source_gradient=None, bilinear=None):
        self._setup(mesh, [HeatTerm(source, fixed_tags, 1.0, source_gradient)], volume, bilinear)

    def _setup(self, mesh, terms, volume, bilinear):
        if mesh.dim != 2:
            raise ConfigError("the heat models are 2D (models/heat.py), as the reference")
        self.space = FunctionSpace(mesh, 1)
        self.material = MaterialIndicator(1.0, CONTRAST)
        if volume <= 0.0:
            raise ConfigError(f"target volume must be positive, got {volume}")
        self.volume = float(volume)
        default_w = 1.0 / len(terms)
        pts = _quad_points(mesh).reshape(-1, 2)
        ne = mesh.num_elements
        area = mesh.measure / ne
        elems = mesh.elements
        self._weights, self._bcs, loads, fq, gq = [], [], [], [], []
        any_grad = any(t.source_gradient is not None for t in terms)
        for t in terms:
            if mesh.facets_with_tag(t.fixed_tags).size == 0:
                raise ConfigError(f"no boundary facets carry ground tags {t.fixed_tags}")
            bc = DirichletSet.on_tags(self.space, t.fixed_tags)
            f_q = np.asarray(t.source(pts), dtype=float).reshape(ne, 3)
            if not np.all(np.isfinite(f_q)):
                raise ConfigError("heat source evaluates to non-finite values")
            # scalar_load (fem.py:414-416): (|T|/3) sum_q f_q N_a(x_q), assembled once
            load = np.zeros(mesh.num_vertices)
            np.add.at(load, elems, (area / 3.0) * (f_q @ _BARY))
            load[bc.dofs] = bc.values
            self._weights.append(default_w if t.weight is None else float(t.weight))
            self._bcs.append(bc)
            loads.append(load)
            fq.append(f_q)
            if any_grad:
                gq.append(np.zeros((ne, 3, 2)) if t.source_gradient is None else
                          np.asarray(t.source_gradient(pts), dtype=float).reshape(ne, 3, 2))
        self._loads = to_device(np.stack(loads))
        self._fq = to_device(np.stack(fq))
        self._gq = to_device(np.stack(gq)) if any_grad else None
        self._has_s0 = any_grad
        # terms grounded on the same tags share one operator (one PCG batch)
        self._groups = {}
        for idx, bc in enumerate(self._bcs):
            self._groups.setdefault(bc.dofs.tobytes(), []).append(idx)
        if bilinear is not None:
            self._bilinear = bilinear
        else:
            self._bilinear = BilinearSpec(stiffness_weight=1.0, boundary_normal_penalty=1e4)
        nparts = int(_lib.load().lsg_partials_per_rhs(mesh.grid)) * 4
        self._partials = torch.zeros(nparts, dtype=torch.float64, device="cuda")
        self._counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._out = torch.zeros(2, dtype=torch.float64, device="cuda")
        self._cache_key = self._cache = None
        self._operators = None

    @property
    def constraint_count(self):
        return 1

    @property
    def load_vectors(self):
        return self._loads

    def operators(self, phi):
        """One Dirichlet-eliminated diffusion operator per ground set (per phi)."""
        if self._operators is None or self._operators[0] is not phi:
            ops = {}
            for key, members in self._groups.items():
                ops[key] = LaplaceOperator(self.space, phi.values, self.material.outside,
                                           self._bcs[members[0]], self.material.inside)
            self._operators = (phi, ops)
        return self._operators[1]

    def pde(self, phi):
        self._check_level(phi)
        ops = self.operators(phi)
        return [LinearProblem(self.space, ops[bc.dofs.tobytes()], self._loads[t], bc)
                for t, bc in enumerate(self._bcs)]

    def adjoint(self, phi, states):
        return [FemField(self.space, -w * u.values) for w, u in zip(self._weights, states)]

    def _evaluate(self, phi, states):
        key = (id(phi), tuple(id(u) for u in states))
        if self._cache_key == key:
            return self._cache
        op = next(iter(self.operators(phi).values()))  # material words are shared
        u = torch.stack([s.values for s in states]).contiguous()
        n = 2 * self.space.mesh.num_vertices
        vc = torch.empty(n, dtype=torch.float64, device="cuda")
        vv = torch.empty(n, dtype=torch.float64, device="cuda")
        wts = np.asarray(self._weights, dtype=np.float64)  # host array, copied into the launch
        _lib.call("lsg_heat_shape", op._op(), int(u.shape[0]), _lib.ptr(u),
                  wts.ctypes.data, _lib.ptr(self._fq), _lib.ptr(self._gq),
                  float(self.volume), _lib.ptr(vc), _lib.ptr(vv), _lib.ptr(self._out),
                  _lib.ptr(self._partials), _lib.ptr(self._counter), _lib.stream())
        J, vol = self._out.tolist()
        self._cache_key = key
        self._cache = (float(J), float(vol), vc, vv)
        return self._cache

    def cost(self, phi, states):
        self._check_level(phi)
        return self._evaluate(phi, states)[0]

    def constraint(self, phi, states):
        return np.array([self._evaluate(phi, states)[1] / self.volume])

    def derivative(self, phi, states, adjoints):
        self._check_level(phi)
        _, _, vc, vv = self._evaluate(phi, states)

        def vol_s1(space):
            chi = phi.indicator_quad()
            return chi[:, :, None, None] * (torch.eye(2, dtype=torch.float64, device="cuda") / self.volume)

        return DerivativePair(vector=((1.0, vc),)), [DerivativePair(s1=vol_s1, vector=((1.0, vv),))]


class HeatPlusModel(HeatModel):
    """Weighted sum of thermal compliances over several terms (``heat.py:165-171``)."""

    def __init__(self, mesh, terms, volume, bilinear=None):
        if len(terms) < 2:
            raise ConfigError("heat sum needs at least two terms; use HeatModel for one")
        self._setup(mesh, list(terms), volume, bilinear)

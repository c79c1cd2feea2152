"""Inclusion recovery from boundary measurements (drop-in for reference ``models/inverse.py``).

Same contract as ``MeasurementPair`` / ``InverseElasticityModel`` /
``dirichlet_extension`` / ``generate_measurements`` (``inverse.py:46-353``):
for every measurement pair two states share one operator -- u driven by the
applied traction (partial clamp) and the lifted correction v in H^1_0
carrying the measured displacement g -- and the Kohn-Vogelius misfit
J = sum_k alpha/2 |u_k - v_k - g_k|^2_D + beta/2 |u_k - g_k|^2_Gamma is the
cost.  States are u_1..u_N then v_1..v_N, adjoints p_1..p_N then q_1..q_N
(``:86-95``); no volume constraint.  The stiff inclusion (contrast kappa) is
the subzero set: A = kappa inside, 1 outside (``:102``).

Device path, per optimisation iteration: the 2N states and the 2N adjoints
are two batched PCG solves each (forced / adjoint-head on the partially
clamped operator, lifted / adjoint-tail on the fully clamped one); the
lifted right-hand sides -K g are one batched apply; the misfit pass
(``lsg_inverse_misfit``) forms the adjoint right-hand sides and J in one
node-gather kernel; ``lsg_inverse_tensors`` evaluates S0 / S1
(``:235-279``), contracted by the velocity solver.  The measured-data
preprocessing (traction loads, the nodal strain projections of g,
``:128-155``) runs once at construction, the projections as batched mass
solves on the device.
"""

from dataclasses import dataclass

import numpy as np
import torch

from .. import _lib
from ..errors import ConfigError
from ..fem import (DirichletSet, ElasticityOperator, FemField, FunctionSpace, H1Operator,
                   LaplaceOperator, LinearProblem, solve_batched, to_device)
from ..velocity import BilinearSpec, DerivativePair
from .base import MaterialIndicator, ModelProblem, as_lame
from .compliance import traction_vector

__all__ = ["MeasurementPair", "InverseElasticityModel", "dirichlet_extension",
           "generate_measurements"]


@dataclass(frozen=True)
class MeasurementPair:
    """One experiment: a traction on a boundary strip and the displacement
    field it produced, already extended into the bulk (``inverse.py:46-54``)."""

    traction: object
    force_tags: object
    measured: FemField


def _tag_tuple(tags):
    if isinstance(tags, (int, np.integer)):
        return (int(tags),)
    return tuple(int(t) for t in tags)


def _assemble_traction(space, tags, traction):
    facets = space.mesh.facets_with_tag(tags)
    if facets.size == 0:
        raise ConfigError(f"no boundary facets carry force tags {tags}")
    if not callable(traction):
        vec = np.asarray(traction, dtype=float)
        if vec.shape != (2,):
            raise ConfigError(f"traction must be a 2-vector, got shape {vec.shape}")
    return traction_vector(space, facets, traction)


def _facet_flags(mesh, facet_ids):
    """Per node: bit 0 = boundary facet (node, node+1), bit 1 = (node, node+nx+1) is listed."""
    nxp = mesh.n[0] + 1
    flags = np.zeros(mesh.num_vertices, dtype=np.uint8)
    f = mesh.boundary_facets[facet_ids]
    a, b = np.minimum(f[:, 0], f[:, 1]), np.maximum(f[:, 0], f[:, 1])
    horiz = (b - a) == 1
    np.bitwise_or.at(flags, a[horiz], np.uint8(1))
    np.bitwise_or.at(flags, a[~horiz], np.uint8(2))
    if not np.all((b - a)[~horiz] == nxp):
        raise ConfigError("boundary facets of a structured mesh join lattice neighbours")
    return to_device(flags, torch.uint8)


class InverseElasticityModel(ModelProblem):
    """Kohn-Vogelius misfit over measurement pairs (``inverse.py:78-279``)."""

    def __init__(self, mesh, fixed_tags, measured_tags, pairs, contrast=10.0, alpha=1.0, beta=1.0,
                 lame=None, bilinear=None):
        if not pairs:
            raise ConfigError("need at least one measurement pair")
        if mesh.dim != 2:
            raise ConfigError("the inverse model is 2D (models/inverse.py), as the reference")
        self.space = FunctionSpace(mesh, 2)
        self.lame = as_lame(lame)
        self.material = MaterialIndicator(contrast, 1.0)
        self.alpha = float(alpha)
        self.beta = float(beta)
        if min(self.alpha, self.beta) < 0.0:
            raise ConfigError("misfit weights must be nonnegative")
        if mesh.facets_with_tag(fixed_tags).size == 0:
            raise ConfigError(f"no boundary facets carry fixed tags {fixed_tags}")
        self.bc_partial = DirichletSet.on_tags(self.space, fixed_tags)
        self.bc_total = DirichletSet.whole_boundary(self.space)
        self.measured_facets = mesh.facets_with_tag(measured_tags)
        if self.measured_facets.size == 0:
            raise ConfigError(f"no boundary facets carry measurement tags {measured_tags}")
        self.pairs = list(pairs)
        loads = []
        for pair in self.pairs:
            g = pair.measured
            if not isinstance(g, FemField) or g.space.value_rank != 2:
                raise ConfigError("measured displacement must be a vector field")
            if g.space.mesh is not mesh:
                raise ConfigError("measured displacement lives on another mesh")
            load = _assemble_traction(self.space, pair.force_tags, pair.traction)
            load[self.bc_partial.dofs] = self.bc_partial.values
            loads.append(load)
        self._loads = to_device(np.stack(loads))
        self._g = torch.stack([to_device(p.measured.values) for p in self.pairs]).contiguous()
        self._flags = _facet_flags(mesh, self.measured_facets)
        self._pmask = self.bc_partial.node_mask(self.space)
        # boundary-zeroing helper: H1 words with the whole-boundary Dirichlet bit
        self._zero_bnd = H1Operator(self.space, 1.0, 0.0, zero_dirichlet=True)
        self._proj = self._project_strains()
        if bilinear is not None:
            self._bilinear = bilinear
        else:
            self._bilinear = BilinearSpec(mass_weight=0.1, stiffness_weight=1.0, zero_dirichlet=True)
        self._partials = torch.zeros(1024, dtype=torch.float64, device="cuda")
        self._counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._out = torch.zeros(1, dtype=torch.float64, device="cuda")
        self._ops = None
        self._misfit_key = self._misfit = None

    def _project_strains(self):
        """Nodal L2 projections of eps_xx, eps_xy, eps_yy of every g (``inverse.py:142-155``):
        P1 mass solves (Jacobi-PCG, the reference's solve_linear) batched over 3 k fields."""
        k, n = self._g.shape
        rhs = torch.empty((k, 3, n), dtype=torch.float64, device="cuda")
        _lib.call("lsg_strain_projection_rhs", self.space.mesh.grid, int(k), _lib.ptr(self._g),
                  _lib.ptr(rhs), _lib.stream())
        mass = H1Operator(self.space, 1.0, 0.0)
        x, _ = solve_batched(mass, rhs.reshape(3 * k, n))
        return x.reshape(k, 3, n).contiguous()

    @property
    def constraint_count(self):
        return 0

    def operators(self, phi):
        """(no clamp, partial clamp, whole-boundary clamp) operators of A(phi)."""
        if self._ops is None or self._ops[0] is not phi:
            mk = lambda bc: ElasticityOperator(self.space, phi.values, self.lame, self.material.outside,
                                               bc, self.material.inside)
            self._ops = (phi, mk(None), mk(self.bc_partial), mk(self.bc_total))
        return self._ops[1:]

    def pde(self, phi):
        self._check_level(phi)
        free, partial, total = self.operators(phi)
        kg = free.apply(self._g)
        lifted = torch.empty_like(kg)
        zero = torch.zeros(kg.shape[1], dtype=torch.float64, device="cuda")
        for r in range(kg.shape[0]):  # -K g, zeroed on the whole boundary (H^1_0 correction)
            _lib.call("lsg_velocity_rhs", self._zero_bnd._op(), _lib.ptr(kg[r]), _lib.ptr(zero), 0.0,
                      _lib.ptr(lifted[r]), _lib.stream())
        k = len(self.pairs)
        forced = [LinearProblem(self.space, partial, self._loads[r], self.bc_partial) for r in range(k)]
        return forced + [LinearProblem(self.space, total, lifted[r], self.bc_total) for r in range(k)]

    def _run_misfit(self, states):
        key = tuple(id(s) for s in states)
        if self._misfit_key == key:
            return self._misfit
        k = len(self.pairs)
        u = torch.stack([s.values for s in states[:k]]).contiguous()
        v = torch.stack([s.values for s in states[k:]]).contiguous()
        head, tail = torch.empty_like(u), torch.empty_like(u)
        _lib.call("lsg_inverse_misfit", self.space.mesh.grid, int(k), _lib.ptr(u), _lib.ptr(v),
                  _lib.ptr(self._g), _lib.ptr(self._flags), _lib.ptr(self._pmask), self.alpha,
                  self.beta, _lib.ptr(head), _lib.ptr(tail), _lib.ptr(self._out),
                  _lib.ptr(self._partials), _lib.ptr(self._counter), _lib.stream())
        self._misfit_key = key
        self._misfit = (float(self._out.item()), head, tail, u, v)
        return self._misfit

    def adjoint(self, phi, states):
        self._check_level(phi)
        _, partial, total = self.operators(phi)
        _, head, tail, _, _ = self._run_misfit(states)
        k = len(self.pairs)
        return ([LinearProblem(self.space, partial, head[r], self.bc_partial) for r in range(k)]
                + [LinearProblem(self.space, total, tail[r], self.bc_total) for r in range(k)])

    def cost(self, phi, states):
        self._check_level(phi)
        return self._run_misfit(states)[0]

    def constraint(self, phi, states):
        return np.zeros(0)

    def tensors(self, phi, states, adjoints):
        """S0 (E,3,2) and S1 (E,3,2,2) of the misfit (``inverse.py:235-279``)."""
        k = len(self.pairs)
        _, _, _, u, v = self._run_misfit(states)
        p = torch.stack([a.values for a in adjoints[:k]]).contiguous()
        q = torch.stack([a.values for a in adjoints[k:]]).contiguous()
        ne = self.space.mesh.num_elements
        s0 = torch.empty((ne, 3, 2), dtype=torch.float64, device="cuda")
        s1 = torch.empty((ne, 3, 2, 2), dtype=torch.float64, device="cuda")
        _lib.call("lsg_inverse_tensors", self.space.mesh.grid, int(k), _lib.ptr(u), _lib.ptr(v),
                  _lib.ptr(p), _lib.ptr(q), _lib.ptr(self._g), _lib.ptr(self._proj),
                  _lib.ptr(phi.values), self.material.inside, self.material.outside,
                  self.lame[0], self.lame[1], self.alpha, _lib.ptr(s0), _lib.ptr(s1), _lib.stream())
        return s0, s1

    def derivative(self, phi, states, adjoints):
        self._check_level(phi)
        s0, s1 = self.tensors(phi, states, adjoints)
        return DerivativePair(s0=lambda space: s0, s1=lambda space: s1), []


def dirichlet_extension(mesh, tags, traces):
    """Harmonic extension of boundary data on the tagged facets (``inverse.py:282-313``):
    componentwise Laplace solves with the trace values on the tagged nodes, all
    components of all traces in one PCG batch."""
    if not traces:
        raise ConfigError("no boundary traces to extend")
    space = traces[0].space
    if space.mesh is not mesh:
        raise ConfigError("traces live on another mesh")
    facets = mesh.facets_with_tag(tags)
    if facets.size == 0:
        raise ConfigError(f"no boundary facets carry tags {tags}")
    for t in traces:
        if t.space is not space:
            raise ConfigError("all traces must share one space")
    nodes = np.unique(mesh.boundary_facets[facets])
    scalar = FunctionSpace(mesh, 1)
    bc = DirichletSet(nodes)
    uniform = -torch.ones(mesh.num_vertices, dtype=torch.float64, device="cuda")  # A = 1 everywhere
    free = LaplaceOperator(scalar, uniform, 1.0)
    clamped = LaplaceOperator(scalar, uniform, 1.0, bc)
    d = space.value_rank
    vals = torch.stack([to_device(t.values).reshape(-1, d).t() for t in traces]).reshape(-1, mesh.num_vertices)
    idx = torch.as_tensor(nodes, device="cuda")
    lift = torch.zeros_like(vals)
    lift[:, idx] = vals[:, idx]
    rhs = -free.apply(lift.contiguous())
    rhs[:, idx] = vals[:, idx]
    x, _ = solve_batched(clamped, rhs.contiguous())
    x = x.reshape(len(traces), d, -1)
    return [FemField(space, x[t].t().contiguous().reshape(-1)) for t in range(len(traces))]


def _vertex_injection(fine_mesh, coarse_mesh):
    """Fine vertex index of every coarse vertex (``inverse.py:316-330``); nested meshes."""
    def keys(pts):
        return np.round(pts * 1e9).astype(np.int64)

    lookup = {tuple(k): i for i, k in enumerate(keys(fine_mesh.vertices))}
    idx = np.empty(coarse_mesh.num_vertices, dtype=np.int64)
    for c, k in enumerate(keys(coarse_mesh.vertices)):
        hit = lookup.get(tuple(k))
        if hit is None:
            raise ConfigError("meshes are not nested: a coarse vertex is missing from the fine mesh")
        idx[c] = hit
    return idx


def generate_measurements(fine_mesh, coarse_mesh, inclusion, forces, fixed_tags, measured_tags,
                          contrast=10.0, lame=None):
    """Twin-experiment data (``inverse.py:333-353``): solve with the true inclusion on
    the fine mesh (one PCG batch over the forces), restrict each displacement to
    the coarse vertices, extend harmonically from the clamp + measured boundary."""
    if not forces:
        raise ConfigError("no forces given")
    injection = _vertex_injection(fine_mesh, coarse_mesh)
    lame = as_lame(lame)
    material = MaterialIndicator(contrast, 1.0)
    fine_scalar = FunctionSpace(fine_mesh, 1)
    level = fine_scalar.interpolate(inclusion)
    fine_space = FunctionSpace(fine_mesh, 2)
    if fine_mesh.facets_with_tag(fixed_tags).size == 0:
        raise ConfigError(f"no boundary facets carry fixed tags {fixed_tags}")
    bc = DirichletSet.on_tags(fine_space, fixed_tags)
    op = ElasticityOperator(fine_space, level.values, lame, material.outside, bc, material.inside)
    loads = []
    for traction, tags in forces:
        load = _assemble_traction(fine_space, tags, traction)
        load[bc.dofs] = bc.values
        loads.append(load)
    fine_u, _ = solve_batched(op, to_device(np.stack(loads)))
    coarse_space = FunctionSpace(coarse_mesh, 2)
    inj = torch.as_tensor(injection, device="cuda")
    injected = [FemField(coarse_space, fine_u[r].reshape(-1, 2)[inj].reshape(-1).contiguous())
                for r in range(len(forces))]
    extended = dirichlet_extension(coarse_mesh, _tag_tuple(fixed_tags) + _tag_tuple(measured_tags),
                                   injected)
    return [MeasurementPair(traction, tags, g) for (traction, tags), g in zip(forces, extended)]

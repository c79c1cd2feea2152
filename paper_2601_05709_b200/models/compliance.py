"""Minimum-compliance models under a volume constraint (drop-in for reference ``models/compliance.py``).

Same contract as ``ComplianceModel`` / ``CompliancePlusModel``
(``compliance.py:37-156``): one shared elasticity operator for every load
(``:97-106``), closed-form adjoint -2u (``:108-109``), J = sum_k int A
sigma_k : eps_k (``:111-123``), C = |{phi<0}| / V (``base.py:150-152``),
S1 = A sum_k (2 G_k^T sigma_k - (sigma_k:eps_k) I) (``:128-139``).

Differences, all additive: ``ersatz`` (the reference hard-codes 1e-4,
``:34``) and ``body_force`` (a constant volume load, as cfg4 needs) are
constructor arguments, and 3D meshes are accepted.

Device path: ``pde`` builds an ``ElasticityOperator`` (one material byte /
word per node); ``cost`` runs the fused compliance + shape-derivative kernel
once and caches J, the volume and the two contracted derivative vectors,
which ``constraint`` and ``derivative`` then reuse -- one pass over the
states per optimisation iteration.
"""

import numpy as np
import torch

from .. import _lib
from ..errors import ConfigError
from ..fem import DirichletSet, ElasticityOperator, FemField, FunctionSpace, LinearProblem, to_device
from ..velocity import BilinearSpec, DerivativePair
from .base import MaterialIndicator, ModelProblem, as_lame

__all__ = ["ComplianceModel", "CompliancePlusModel", "ERSATZ", "traction_vector",
           "body_force_vector"]

ERSATZ = 1e-4


def traction_vector(space, facet_ids, g):
    """Load vector of a constant traction g on boundary facets (``fem.py:441-448``).

    2D keeps the reference's 2-point Gauss rule on each facet; 3D integrates
    the P1 basis exactly on each triangle facet (|f|/3 per vertex).  Setup
    only (a few facets), assembled on the host.
    """
    mesh = space.mesh
    d = mesh.dim
    facets = mesh.boundary_facets[facet_ids]
    meas = mesh.facet_measures[facet_ids]
    if callable(g):  # sampled at the facet Gauss points (boundary_vector_load, fem.py:441-448)
        if d != 2:
            raise ConfigError("callable tractions are 2D only, as the reference")
        gp = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
        a, b = mesh.vertices[facets[:, 0]], mesh.vertices[facets[:, 1]]
        pts = a[:, None, :] + gp[None, :, None] * (b - a)[:, None, :]
        g_q = np.asarray(g(pts), dtype=float).reshape(len(facets), 2, 2)
    else:
        g = np.asarray(g, dtype=float)
        if g.shape != (d,):
            raise ConfigError(f"traction must be a {d}-vector, got shape {g.shape}")
        g_q = np.broadcast_to(g, (len(facets), 2, d))
    if d == 2:
        gp = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
        basis = np.stack([1.0 - gp, gp], axis=1)
        w = np.repeat((meas / 2.0)[:, None], 2, axis=1)
        elems = np.einsum("fqc,qa->fac", w[:, :, None] * g_q, basis)
    else:
        elems = np.broadcast_to((meas / 3.0)[:, None, None] * g[None, None, :], (len(facets), 3, 3))
    out = np.zeros(space.dof_count)
    dofs = d * facets[:, :, None] + np.arange(d)[None, None, :]
    np.add.at(out, dofs.reshape(len(facets), -1), elems.reshape(len(facets), -1))
    return out


def _lumped_counts(mesh):
    """Number of elements containing each node, closed form on the lattice."""
    n = mesh.n
    if mesh.dim == 2:
        nx, ny = n
        c = np.zeros((ny + 1, nx + 1))
        c[:-1, :-1] += 2  # cell (i, j): lower a + upper a
        c[:-1, 1:] += 1   # cell (i-1, j): lower b
        c[1:, :-1] += 1   # cell (i, j-1): upper d
        c[1:, 1:] += 2    # cell (i-1, j-1): lower c + upper c
        return c.reshape(-1)
    nx, ny, nz = n
    c = np.zeros((nz + 1, ny + 1, nx + 1))
    for dz in (0, 1):
        for dy in (0, 1):
            for dx in (0, 1):
                corner = (dx, dy, dz)
                cnt = 6 if corner in ((0, 0, 0), (1, 1, 1)) else 2
                c[dz:dz + nz, dy:dy + ny, dx:dx + nx] += cnt
    return c.reshape(-1)


def body_force_vector(space, f):
    """Exact P1 load of a constant body force f: (|T|/(d+1)) f per element vertex
    (``vector_load``, ``fem.py:419-425``)."""
    mesh = space.mesh
    d = mesh.dim
    f = np.asarray(f, dtype=float)
    cell = mesh.measure / mesh.num_elements
    w = _lumped_counts(mesh) * (cell / (d + 1))
    return (w[:, None] * f[None, :]).reshape(-1)


class ComplianceModel(ModelProblem):
    """Single traction load: J = int A sigma(u) : eps(u) (``compliance.py:37-133``)."""

    def __init__(self, mesh, fixed_tags, load_tags, traction, volume, lame=None, frozen=None,
                 bilinear=None, ersatz=ERSATZ, body_force=None):
        self._setup(mesh, fixed_tags, [(traction, load_tags)] if traction is not None else [],
                    volume, lame, frozen, bilinear, ersatz, body_force)

    def _setup(self, mesh, fixed_tags, loads, volume, lame, frozen, bilinear, ersatz=ERSATZ,
               body_force=None):
        self.space = FunctionSpace(mesh, mesh.dim)
        self.lame = as_lame(lame)
        self.material = MaterialIndicator(1.0, float(ersatz))
        if volume <= 0.0:
            raise ConfigError(f"target volume must be positive, got {volume}")
        self.volume = float(volume)
        if mesh.facets_with_tag(fixed_tags).size == 0:
            raise ConfigError(f"no boundary facets carry fixed tags {fixed_tags}")
        self.bc = DirichletSet.on_tags(self.space, fixed_tags)
        vectors = []
        for traction, tags in loads:
            facets = mesh.facets_with_tag(tags)
            if facets.size == 0:
                raise ConfigError(f"no boundary facets carry load tags {tags}")
            vectors.append(traction_vector(self.space, facets, traction))
        if body_force is not None:
            bf = body_force_vector(self.space, body_force)
            vectors = [v + bf for v in vectors] if vectors else [bf]
        if not vectors:
            raise ConfigError("compliance model needs at least one load")
        for v in vectors:  # Dirichlet rows of the eliminated system carry the values (0)
            v[self.bc.dofs] = self.bc.values
        self._loads = to_device(np.stack(vectors))
        if bilinear is not None:
            self._bilinear = bilinear
        else:
            self._bilinear = BilinearSpec(
                mass_weight=0.1, stiffness_weight=1.0, boundary_normal_penalty=1e4,
                frozen_subdomain=frozen, frozen_penalty=1e4 if frozen is not None else 0.0)
        self._cache_key = None
        self._cache = None
        nparts = int(_lib.load().lsg_partials_per_rhs(mesh.grid)) * 4
        self._partials = torch.zeros(nparts, dtype=torch.float64, device="cuda")
        self._counter = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._out = torch.zeros(2, dtype=torch.float64, device="cuda")
        self._operator = None

    @property
    def load_vectors(self):
        return self._loads

    @property
    def constraint_count(self):
        return 1

    # -- contract --------------------------------------------------------------------
    def operator(self, phi):
        if self._operator is None or self._operator[0] is not phi:
            op = ElasticityOperator(self.space, phi.values, self.lame,
                                    self.material.outside, self.bc, self.material.inside)
            self._operator = (phi, op)
        return self._operator[1]

    def pde(self, phi):
        self._check_level(phi)
        op = self.operator(phi)
        return [LinearProblem(self.space, op, self._loads[k], self.bc)
                for k in range(self._loads.shape[0])]

    def adjoint(self, phi, states):
        return [FemField(self.space, -2.0 * u.values) for u in states]

    def _evaluate(self, phi, states):
        key = (id(phi), tuple(id(u) for u in states))
        if self._cache_key == key:
            return self._cache
        op = self.operator(phi)
        u = torch.stack([s.values for s in states]).contiguous()
        n = self.space.dof_count
        vc = torch.empty(n, dtype=torch.float64, device="cuda")
        vv = torch.empty(n, dtype=torch.float64, device="cuda")
        _lib.call("lsg_shape_rhs", op._op(), int(u.shape[0]), _lib.ptr(u), float(self.volume),
                  _lib.ptr(vc), _lib.ptr(vv), _lib.ptr(self._out), None, _lib.ptr(self._partials),
                  _lib.ptr(self._counter), _lib.stream())
        J, vol = self._out.tolist()
        self._cache_key = key
        self._cache = (float(J), float(vol), vc, vv, u)
        return self._cache

    def cost(self, phi, states):
        self._check_level(phi)
        return self._evaluate(phi, states)[0]

    def constraint(self, phi, states):
        return np.array([self._evaluate(phi, states)[1] / self.volume])

    def s1_tensor(self, phi, states):
        """S1 of the cost per element and quadrature point (parity path)."""
        op = self.operator(phi)
        u = torch.stack([s.values for s in states]).contiguous()
        nq = 3 if self.space.dim == 2 else 4
        d = self.space.dim
        s1 = torch.empty((self.space.mesh.num_elements, nq, d, d), dtype=torch.float64, device="cuda")
        _lib.call("lsg_s1_tensor", op._op(), int(u.shape[0]), _lib.ptr(u), _lib.ptr(phi.values),
                  _lib.ptr(s1), _lib.stream())
        return s1

    def derivative(self, phi, states, adjoints):
        self._check_level(phi)
        _, _, vc, vv, _ = self._evaluate(phi, states)
        d = self.space.dim
        cost_pair = DerivativePair(s1=lambda space: self.s1_tensor(phi, states), vector=((1.0, vc),))

        def vol_s1(space):
            chi = phi.indicator_quad()
            return chi[:, :, None, None] * (torch.eye(d, dtype=torch.float64, device="cuda") / self.volume)

        return cost_pair, [DerivativePair(s1=vol_s1, vector=((1.0, vv),))]


class CompliancePlusModel(ComplianceModel):
    """Sum of compliances over several loads (``compliance.py:142-156``); all
    load cases are solved as one batch."""

    def __init__(self, mesh, fixed_tags, loads, volume, lame=None, frozen=None, bilinear=None,
                 ersatz=ERSATZ, body_force=None):
        if len(loads) < 2:
            raise ConfigError("compliance sum needs at least two loads; use ComplianceModel for a single one")
        self._setup(mesh, fixed_tags, list(loads), volume, lame, frozen, bilinear, ersatz, body_force)

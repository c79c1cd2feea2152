"""P1 spaces, matrix-free operators and the batched Jacobi-PCG (drop-in for reference ``fem.py``).

* ``FunctionSpace`` / ``FemField`` keep the reference's dof convention
  (dof = d*node + c, ``fem.py:56-96``); field values are fp64 CUDA tensors.
* ``DirichletSet`` mirrors ``fem.py:213-266``; on the device it becomes one
  bit per dof in the operator's per-node word.
* ``ElasticityOperator`` replaces the assembled CSR matrix of
  ``elasticity_matrix`` + ``assemble_matrix`` (``fem.py:397-411, 141-150``):
  it holds only the per-node material word (1 byte/node in 2D) computed from
  the level set; ``apply`` is the warp-marching stencil kernel.
* ``solve_linear`` / ``solve_batched`` replace scipy ``cg`` with the Jacobi
  preconditioner (``fem.py:294-316``), same stopping rule
  ``||r|| < max(atol, rtol ||b||)``, same iteration cap 10n and the same
  ``SolverError(residual)``; k right-hand sides sharing one operator run as
  one batched launch (replacing the thread pool of ``driver.py:169-194``).
"""

import itertools

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, SolverError

__all__ = ["FunctionSpace", "FemField", "DirichletSet", "ElasticityOperator", "H1Operator", "LaplaceOperator",
           "LinearProblem", "solve_linear", "solve_batched", "CG_RTOL", "CG_ATOL",
           "CG_ITER_FACTOR", "to_device"]

CG_RTOL = 1e-10
CG_ATOL = 1e-14
CG_ITER_FACTOR = 10

# When set to a list, solve_batched appends one record per launched PCG chunk
# (CUDA events around lsg_pcg_iterate + completed iterations): bench.py uses
# it to time the fused PCG iteration live, on the launching stream.
PCG_PROFILE = None


def to_device(values, dtype=torch.float64):
    if isinstance(values, torch.Tensor):
        return values.to(device="cuda", dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(values), dtype=dtype, device="cuda")


class FunctionSpace:
    """Nodal P1 space of value rank 1 (scalar) or dim (vector) on a structured mesh."""

    def __init__(self, mesh, value_rank=1):
        if value_rank not in (1, mesh.dim):
            raise ConfigError(f"value_rank must be 1 or {mesh.dim}, got {value_rank}")
        self.mesh = mesh
        self.value_rank = value_rank

    @property
    def dim(self):
        return self.mesh.dim

    @property
    def dof_count(self):
        return self.mesh.num_vertices * self.value_rank

    def zero_field(self):
        return FemField(self, torch.zeros(self.dof_count, dtype=torch.float64, device="cuda"))

    def interpolate(self, fn):
        """Nodal interpolation of ``fn(points) -> (N,) or (N, d)`` (``fem.py:103-112``)."""
        vals = np.asarray(fn(self.mesh.vertices), dtype=float)
        if self.value_rank == 1:
            if vals.shape != (self.mesh.num_vertices,):
                raise ConfigError(f"scalar interpolant has shape {vals.shape}")
        elif vals.shape != (self.mesh.num_vertices, self.value_rank):
            raise ConfigError(f"vector interpolant has shape {vals.shape}")
        return FemField(self, to_device(vals.reshape(-1)))


class FemField:
    """Nodal coefficients (fp64 CUDA tensor) tied to their space."""

    def __init__(self, space, values):
        self.space = space
        self.values = to_device(values)
        if self.values.shape != (space.dof_count,):
            raise ConfigError(f"field has shape {tuple(self.values.shape)}, expected ({space.dof_count},)")

    def copy(self):
        return FemField(self.space, self.values.clone())

    def numpy(self):
        return self.values.detach().cpu().numpy()


class DirichletSet:
    """Constrained dofs with prescribed values (``fem.py:213-266``)."""

    def __init__(self, dofs, values=None):
        dofs = np.asarray(dofs, dtype=np.int64)
        if values is None:
            values = np.zeros(len(dofs))
        values = np.broadcast_to(np.asarray(values, dtype=float), dofs.shape)
        order = np.argsort(dofs, kind="stable")
        d, v = dofs[order], values[order]
        uniq, first = np.unique(d, return_index=True)
        ref = v[first][np.searchsorted(uniq, d)]
        if np.any(ref != v):
            raise ConfigError(f"conflicting Dirichlet values for dofs {d[ref != v][:5]}")
        self.dofs = uniq
        self.values = v[first]

    def __len__(self):
        return len(self.dofs)

    def homogeneous(self):
        return DirichletSet(self.dofs, np.zeros(len(self.dofs)))

    @staticmethod
    def on_tags(space, tags, value=0.0):
        facet_ids = space.mesh.facets_with_tag(tags)
        nodes = np.unique(space.mesh.boundary_facets[facet_ids])
        d = space.value_rank
        if callable(value):
            vals = np.asarray(value(space.mesh.node_coords(nodes)), dtype=float)
        else:
            shape = (len(nodes),) if d == 1 else (len(nodes), d)
            vals = np.broadcast_to(float(value), shape)
        if d == 1:
            return DirichletSet(nodes, vals)
        dofs = (d * nodes[:, None] + np.arange(d)[None, :]).reshape(-1)
        return DirichletSet(dofs, np.asarray(vals).reshape(-1))

    @staticmethod
    def whole_boundary(space, value=0.0):
        return DirichletSet.on_tags(space, np.unique(space.mesh.facet_tags), value)

    def node_mask(self, space):
        """Per-node byte, bit c set when dof d*node+c is constrained (device tensor)."""
        d = space.value_rank
        mask = np.zeros(space.mesh.num_vertices, dtype=np.uint8)
        if len(self.dofs):
            np.bitwise_or.at(mask, self.dofs // d, (1 << (self.dofs % d)).astype(np.uint8))
        return to_device(mask, torch.uint8)


class _Operator:
    """Matrix-free operator on a vector space: the ``matrix`` slot of a problem."""

    kind = None
    scalar = False  # True for operators on scalar (temperature) spaces

    def __init__(self, space):
        if space.value_rank != (1 if self.scalar else space.dim):
            raise ConfigError("this operator acts on " + ("scalar" if self.scalar else "vector") + " spaces")
        self.space = space
        self.grid = space.mesh.grid

    @property
    def shape(self):
        n = self.space.dof_count
        return (n, n)

    def _op(self):
        raise NotImplementedError

    def apply(self, x, k=None):
        """y = A x for one field (n,) or a batch (k, n) of fields."""
        x = to_device(x)
        kk = 1 if x.dim() == 1 else x.shape[0]
        y = torch.empty_like(x)
        _lib.call("lsg_apply", self._op(), int(kk), _lib.ptr(x), _lib.ptr(y), _lib.stream())
        return y

    __matmul__ = apply

    def diagonal(self):
        d = torch.empty(self.space.dof_count, dtype=torch.float64, device="cuda")
        _lib.call("lsg_diag", self._op(), _lib.ptr(d), _lib.stream())
        return d

    def inverse_diagonal(self):
        """Jacobi preconditioner diag(1/D) (``fem.py:303-305``), computed once per operator."""
        dinv = getattr(self, "_dinv", None)
        if dinv is None:
            dinv = torch.empty(self.space.dof_count, dtype=torch.float64, device="cuda")
            _lib.call("lsg_inv_diag", self._op(), _lib.ptr(dinv), _lib.stream())
            self._dinv = dinv
        return dinv


class ElasticityOperator(_Operator):
    """Ersatz-material elasticity, Dirichlet-eliminated (``fem.py:397-411, 274-291``).

    ``phi`` is the nodal level set (CUDA tensor); the material word of every
    node is computed once here and reused by every apply of this operator.
    """

    kind = _lib.LSG_OP_ELASTICITY

    def __init__(self, space, phi_values, lame, ersatz, bc=None, inside=1.0):
        super().__init__(space)
        self.lame = (float(lame[0]), float(lame[1]))
        self.ersatz = float(ersatz)
        self.inside = float(inside)
        self.bc = bc
        self.bcmask = bc.node_mask(space) if bc is not None and len(bc) else None
        word_dtype = torch.uint8 if space.dim == 2 else torch.int32
        self.words = torch.empty(space.mesh.num_vertices, dtype=word_dtype, device="cuda")
        phi_values = to_device(phi_values)
        _lib.call("lsg_material", self.grid, _lib.ptr(phi_values), _lib.ptr(self.bcmask),
                  _lib.ptr(self.words), _lib.stream())
        self._cop = _lib.make_op(self.kind, self.grid, self.words,
                                 (self.lame[0], self.lame[1], self.ersatz, self.inside))

    def _op(self):
        return self._cop


class LaplaceOperator(_Operator):
    """Two-phase diffusion (A grad u, grad v) of the heat models, Dirichlet-eliminated
    (``models/heat.py:113-119``, ``fem.py:388-394``); A = inside where phi < 0 at a
    quadrature point, ``contrast`` elsewhere, averaged per triangle.  2D only, as
    the reference."""

    kind = _lib.LSG_OP_LAPLACE
    scalar = True

    def __init__(self, space, phi_values, contrast, bc=None, inside=1.0):
        super().__init__(space)
        if space.dim != 2:
            raise ConfigError("the heat models are 2D (models/heat.py), as the reference")
        self.contrast = float(contrast)
        self.inside = float(inside)
        self.bc = bc
        self.bcmask = bc.node_mask(space) if bc is not None and len(bc) else None
        self.words = torch.empty(space.mesh.num_vertices, dtype=torch.uint8, device="cuda")
        _lib.call("lsg_material", self.grid, _lib.ptr(to_device(phi_values)), _lib.ptr(self.bcmask),
                  _lib.ptr(self.words), _lib.stream())
        self._cop = _lib.make_op(self.kind, self.grid, self.words, (self.contrast, self.inside))

    def _op(self):
        return self._cop


class H1Operator(_Operator):
    """Velocity form B = mw M + sw K + np * normal mass + fp * frozen mass (``velocity.py:98-127``)."""

    kind = _lib.LSG_OP_H1

    def __init__(self, space, mass_weight, stiffness_weight, boundary_normal_penalty=0.0,
                 frozen_q=None, frozen_penalty=0.0, zero_dirichlet=False):
        super().__init__(space)
        word_dtype = torch.uint8 if space.dim == 2 else torch.int32
        self.words = torch.empty(space.mesh.num_vertices, dtype=word_dtype, device="cuda")
        fq = None if frozen_q is None else to_device(np.asarray(frozen_q, dtype=np.uint8), torch.uint8)
        _lib.call("lsg_h1_words", self.grid, _lib.ptr(fq), int(bool(zero_dirichlet)),
                  _lib.ptr(self.words), _lib.stream())
        self.zero_dirichlet = bool(zero_dirichlet)
        self._cop = _lib.make_op(self.kind, self.grid, self.words,
                                 (mass_weight, stiffness_weight, boundary_normal_penalty,
                                  frozen_penalty))

    def _op(self):
        return self._cop


class LinearProblem:
    """One linear state or adjoint system (``models/base.py:42-53``); ``matrix``
    is a matrix-free operator already carrying the elimination of ``bc``."""

    def __init__(self, space, matrix, rhs, bc=None):
        self.space = space
        self.matrix = matrix
        self.rhs = to_device(rhs)
        self.bc = bc


class _Workspace:
    """Device buffers of one batched PCG, cached per (operator grid, k)."""

    def __init__(self, grid, n, k):
        self.k = k
        self.n = n
        dev = dict(dtype=torch.float64, device="cuda")
        self.x = torch.zeros((k, n), **dev)
        self.b = torch.zeros((k, n), **dev)
        self.r = torch.empty((k, n), **dev)
        self.p = torch.empty((k, n), **dev)
        self.q = torch.empty((k, n), **dev)
        self.p_alt = torch.empty((k, n), **dev)
        self.p_ring = torch.empty((k, n), **dev) if grid.dim == 3 else torch.empty(0, **dev)
        self.r_alt = torch.empty((k, n), **dev) if grid.dim == 2 else torch.empty(0, **dev)
        self.q_alt = torch.empty((k, n), **dev) if grid.dim == 2 else torch.empty(0, **dev)
        self.scal = torch.zeros((k, _lib.SCAL_DOUBLES), **dev)
        npart = int(_lib.load().lsg_partials_per_rhs(grid))
        self.partials = torch.zeros(k * npart * 8, **dev)
        self.counters = torch.zeros(max(k, 1), dtype=torch.int32, device="cuda")
        self.host_scal = torch.zeros((k, _lib.SCAL_DOUBLES), dtype=torch.float64, pin_memory=True)
        self.ws = _lib.PcgWs()
        self.ws.k = k
        for name in ("x", "b", "r", "p", "q", "scal", "partials", "counters", "p_alt", "p_ring",
                     "r_alt", "q_alt"):
            setattr(self.ws, name, getattr(self, name).data_ptr())


def _workspace(op, k):
    """The PCG workspace of k right-hand sides on op's mesh.  Cached on the mesh object
    (freed with it; never shared between meshes, dimensions or system sizes)."""
    mesh = op.space.mesh
    key = ("pcg_ws", mesh.dim, mesh.n, op.space.dof_count, k)
    ws = mesh.device_cache.get(key)
    if ws is None:
        ws = _Workspace(op.grid, op.space.dof_count, k)
        mesh.device_cache[key] = ws
    return ws


def _scal(ws, field):
    return ws.host_scal[:, _lib.SCAL_FIELDS.index(field)]


# Iterations the previous solve of the same kind of system needed (max over its
# right-hand sides): the optimisation loop solves warm-started systems whose
# counts change slowly, so the next solve is enqueued as one chunk of ~90% of
# that count and then short chunks, instead of doubling chunks that overshoot
# convergence by up to one chunk of no-op iterations and poll the host ~8 times
# (a chunk is enqueued as power-of-two launches without polling in between).
# Chunking never changes the iterates (the device decides convergence per
# iteration); it only sets how often the host polls.
_LAST_ITERS = {}  # (kind, dim, grid shape, n, k, rtol) -> iterations of the last solve


def _pieces(total):
    """A chunk as power-of-two launches of 32..512 iterations (the CUDA-graph cache
    keys on the iteration count, so only five shapes are ever captured)."""
    out = []
    while total >= 32:
        p = 512
        while p > total:
            p //= 2
        out.append(p)
        total -= p
    return out or [32]


def _chunks(last):
    """Chunk sizes for a solve whose predecessor needed `last` iterations."""
    if not last:
        c = 32
        while True:
            yield c
            c = min(2 * c, 512)
    first = max(32, int(0.9 * last))
    yield first
    step = max(32, last // 16)
    done = first
    while done < 1.5 * last:
        yield step
        done += step
    c = step
    while True:  # far beyond the previous count: back to doubling
        c = min(2 * c, 512)
        yield c


def solve_batched(op, rhs, x0=None, rtol=CG_RTOL, atol=CG_ATOL, maxiter=None, chunk=None):
    """Jacobi-PCG on k right-hand sides sharing ``op``; returns (x (k, n), iterations (k,)).

    scipy ``cg`` semantics per right-hand side: threshold max(atol, rtol ||b||),
    checked before every iteration; b = 0 returns zeros; maxiter defaults to
    10 n; exhaustion raises SolverError carrying the true residual norm.
    """
    b = to_device(rhs)
    if b.dim() == 1:
        b = b[None]
    k, n = b.shape
    ws = _workspace(op, k)
    ws.b.copy_(b)
    if x0 is None:
        ws.x.zero_()
    else:
        x0 = to_device(x0)
        ws.x.copy_(x0.reshape(k, n))
    maxiter = CG_ITER_FACTOR * n if maxiter is None else int(maxiter)
    cop = op._op()
    st = _lib.stream()
    dinv = op.inverse_diagonal()
    ws.ws.dinv = dinv.data_ptr()
    _lib.call("lsg_pcg_start", cop, ws.ws, float(rtol), float(atol), float(maxiter), st)
    stream = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ws.host_scal.copy_(ws.scal, non_blocking=True)
    ev.record(stream)
    ev.synchronize()
    done = _scal(ws, "done")
    prof = PCG_PROFILE
    key = (op.kind, op.space.mesh.dim, op.space.mesh.n, n, k, float(rtol))
    if chunk is not None:
        plan = itertools.repeat(int(chunk))
    else:
        plan = _chunks(_LAST_ITERS.get(key))
    while not bool((done != 0).all()):
        chunk = next(plan)
        if prof is not None:
            before = _scal(ws, "iters").clone()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        for piece in _pieces(chunk):  # power-of-two launches: a handful of graph shapes
            _lib.call("lsg_pcg_iterate", cop, ws.ws, int(piece), st)
        if prof is not None:
            e1.record(stream)
        ws.host_scal.copy_(ws.scal, non_blocking=True)
        ev.record(stream)
        ev.synchronize()
        done = _scal(ws, "done")
        if prof is not None:
            delta = _scal(ws, "iters") - before
            prof.append(dict(kind=op.kind, k=k, n=n, events=(e0, e1), launched=int(chunk),
                             rhs_iters=float(delta.sum()), max_iters=float(delta.max())))
    _lib.call("lsg_pcg_finish", cop, ws.ws, st)  # pending x += alpha p of the last iteration
    iters = _scal(ws, "iters").to(torch.int64).clone()
    _LAST_ITERS[key] = int(iters.max())
    failed = (done == 2).nonzero().flatten().tolist()
    x = ws.x.clone()
    if failed:
        i = failed[0]
        res = float(torch.linalg.vector_norm(b[i] - op.apply(x[i])))
        raise SolverError(f"conjugate gradients stopped after {int(iters[i])} iterations, "
                          f"residual {res:.3e}", residual=res)
    return x, iters


def solve_linear(problem, x0=None, rtol=CG_RTOL):
    """Solve one problem (``fem.py:294-316``); returns the solution tensor."""
    x, _ = solve_batched(problem.matrix, problem.rhs, None if x0 is None else to_device(x0)[None],
                         rtol=rtol)
    return x[0]

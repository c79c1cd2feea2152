"""P1 finite elements on structured simplex meshes (oracle; test infrastructure only).

Restates reference ``fem.py`` for d = 2 (and, as a new dimension-generic
extension, d = 3):

* vector dofs interleave components, dof = d*node + c (``fem.py:56-96``);
* element gradients from the inverse-transposed affine map (``fem.py:62-78``);
* quadrature: 2D edge midpoints of (0,1), (1,2), (0,2) with weights |T|/3
  (``fem.py:42-45,78-80``); 3D the symmetric degree-2 4-point rule with
  weights |T|/4 (same exactness for P1 x P1 products);
* element kernels for mass, Laplace and elasticity (``fem.py:379-411``),
  COO -> CSR assembly (``fem.py:141-155``), symmetric Dirichlet elimination
  (``fem.py:274-291``) and Jacobi-PCG through scipy ``cg`` with rtol 1e-10,
  atol 1e-14, maxiter 10 n (``fem.py:51-53,294-316``).
"""

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

CG_RTOL = 1e-10
CG_ATOL = 1e-14
CG_ITER_FACTOR = 10

QUAD_BARY_2D = np.array([[0.5, 0.5, 0.0], [0.0, 0.5, 0.5], [0.5, 0.0, 0.5]])
TET_A = 0.5854101966249685
TET_B = 0.1381966011250105
QUAD_BARY_3D = np.full((4, 4), TET_B) + np.eye(4) * (TET_A - TET_B)


def quad_bary(dim):
    return QUAD_BARY_2D if dim == 2 else QUAD_BARY_3D


class SolverError(RuntimeError):
    def __init__(self, message, residual=None):
        super().__init__(message)
        self.residual = residual


class Space:
    """Nodal P1 space of value rank 1 (scalar) or d (vector) on a Grid."""

    def __init__(self, grid, value_rank=1):
        assert value_rank in (1, grid.dim)
        self.grid = grid
        self.dim = grid.dim
        self.value_rank = value_rank
        p = grid.vertices[grid.elements]  # (E, d+1, d)
        jac = np.swapaxes(p[:, 1:] - p[:, :1], 1, 2)  # columns = edge vectors
        inv_t = np.linalg.inv(jac).transpose(0, 2, 1)  # (E, d, d)
        ref = np.vstack([-np.ones(self.dim), np.eye(self.dim)])  # (d+1, d)
        self.grads = np.einsum("tdk,ik->tid", inv_t, ref)
        self.measures = grid.element_measures()
        self.bary = quad_bary(self.dim)
        nq = self.bary.shape[0]
        self.quad_weights = np.repeat((self.measures / nq)[:, None], nq, axis=1)
        self.quad_points = np.einsum("qi,tid->tqd", self.bary, p)

    @property
    def dof_count(self):
        return self.grid.num_vertices * self.value_rank

    def element_dofs(self):
        el = self.grid.elements[getattr(self, "sl", slice(None))]
        if self.value_rank == 1:
            return el
        d = self.value_rank
        return (d * el[:, :, None] + np.arange(d)[None, None, :]).reshape(len(el), -1)

    def nodal(self, values):
        values = np.asarray(values)
        if self.value_rank == 1:
            return values[self.grid.elements]
        return values.reshape(-1, self.value_rank)[self.grid.elements]

    def grad_at_quad(self, values):
        """Per-element gradients; vector: result[t, a, b] = d u_a / d x_b."""
        nodal = self.nodal(values)
        if self.value_rank == 1:
            return np.einsum("tid,ti->td", self.grads, nodal)
        return np.einsum("tia,tib->tab", nodal, self.grads)

    def assemble_matrix(self, elems):
        dofs = self.element_dofs()
        rows = np.broadcast_to(dofs[:, :, None], elems.shape)
        cols = np.broadcast_to(dofs[:, None, :], elems.shape)
        n = self.dof_count
        return sp.coo_matrix((elems.ravel(), (rows.ravel(), cols.ravel())), shape=(n, n)).tocsr()

    def part(self, sl):
        """The elements ``sl`` of this space as a space of its own (same dofs):
        what the element-matrix builders read, restricted to a slice."""
        view = object.__new__(Space)
        view.grid, view.dim, view.value_rank, view.bary = self.grid, self.dim, self.value_rank, self.bary
        view.grads, view.measures = self.grads[sl], self.measures[sl]
        view.quad_weights, view.quad_points = self.quad_weights[sl], self.quad_points[sl]
        view.sl = sl
        return view

    def assemble_matrix_by_parts(self, builder, chunk=400_000):
        """assemble_matrix(builder(space)) with the element matrices built and
        summed ``chunk`` elements at a time (cfg5 at full size: 10.6M tets x
        12 x 12 entries do not fit in memory at once).  ``builder`` receives a
        space restricted to a slice (``part.sl``)."""
        nt = len(self.grid.elements)
        out = None
        for start in range(0, nt, chunk):
            view = self.part(slice(start, min(start + chunk, nt)))
            mat = view.assemble_matrix(builder(view))
            out = mat if out is None else out + mat
        return out

    def assemble_vector(self, elems):
        out = np.zeros(self.dof_count)
        np.add.at(out, self.element_dofs(), elems)
        return out


def phi_at_quad_sign(space, phi):
    """Indicator [phi(x_q) < 0] at quadrature points, shape (E, nq).

    2D: phi(x_q) = 0.5 phi_i + 0.5 phi_j (+ 0 phi_k), whose sign equals the
    sign of phi_i + phi_j exactly (reference ``levelset.py:65-67`` evaluates
    the same barycentric sum).  3D: phi(x_q) = ((A phi_q + B phi_o1) + B phi_o2)
    + B phi_o3 with the other three local vertices in ascending order, every
    operation rounded separately (the CUDA kernel uses __dmul_rn/__dadd_rn in
    the same order).
    """
    nodal = np.asarray(phi)[space.grid.elements]
    if space.dim == 2:
        pairs = ((0, 1), (1, 2), (0, 2))
        return np.stack([(0.5 * nodal[:, i] + 0.5 * nodal[:, j]) < 0.0 for i, j in pairs], axis=1)
    cols = []
    for q in range(4):
        others = [i for i in range(4) if i != q]
        v = TET_A * nodal[:, q]
        for o in others:
            v = v + TET_B * nodal[:, o]
        cols.append(v < 0.0)
    return np.stack(cols, axis=1)


def mass_elements(space, coeff_q=None):
    w = space.quad_weights if coeff_q is None else space.quad_weights * coeff_q
    scalar = np.einsum("tq,qa,qb->tab", w, space.bary, space.bary)
    return _expand(space, scalar)


def stiffness_elements(space, coeff_q=None):
    w = (space.quad_weights if coeff_q is None else space.quad_weights * coeff_q).sum(axis=1)
    scalar = np.einsum("t,tad,tbd->tab", w, space.grads, space.grads)
    return _expand(space, scalar)


def _expand(space, scalar):
    if space.value_rank == 1:
        return scalar
    d = space.value_rank
    nt, nl = scalar.shape[:2]
    return np.einsum("tab,ij->taibj", scalar, np.eye(d)).reshape(nt, nl * d, nl * d)


def elasticity_elements(space, coeff_q, lame):
    """(c sigma(u), eps(v)) element matrices, reference ``fem.py:397-411``."""
    lam, mu = lame
    d = space.dim
    w = (space.quad_weights * coeff_q).sum(axis=1)
    g = space.grads
    dot = np.einsum("tad,tbd->tab", g, g)
    inner = (lam * np.einsum("tai,tbj->taibj", g, g)
             + mu * np.einsum("tab,ij->taibj", dot, np.eye(d))
             + mu * np.einsum("taj,tbi->taibj", g, g))
    nt, nl = g.shape[:2]
    return w[:, None, None] * inner.reshape(nt, nl * d, nl * d)


def dirichlet_eliminate(matrix, rhs, dofs, values=None):
    """Symmetric elimination (reference ``fem.py:274-291``)."""
    dofs = np.asarray(dofs, dtype=np.int64)
    if len(dofs) == 0:
        return matrix, rhs
    values = np.zeros(len(dofs)) if values is None else np.asarray(values, dtype=float)
    n = matrix.shape[0]
    constrained = np.zeros(n, dtype=bool)
    constrained[dofs] = True
    lifted = np.zeros(n)
    lifted[dofs] = values
    rhs = rhs - matrix @ lifted
    rhs[dofs] = values
    A = matrix.tocoo()
    keep = ~(constrained[A.row] | constrained[A.col])
    rows = np.concatenate([A.row[keep], dofs])
    cols = np.concatenate([A.col[keep], dofs])
    data = np.concatenate([A.data[keep], np.ones(len(dofs))])
    return sp.coo_matrix((data, (rows, cols)), shape=(n, n)).tocsr(), rhs


def jacobi_pcg(A, b, x0=None, rtol=CG_RTOL, atol=CG_ATOL, maxiter=None):
    """scipy ``cg`` with the Jacobi preconditioner, reference ``fem.py:294-316``.

    Returns (x, iterations).  Raises SolverError(residual) on non-convergence.
    """
    n = A.shape[0]
    diag = A.diagonal()
    safe = np.where(np.abs(diag) > 0.0, diag, 1.0)
    M = sp.diags(1.0 / safe)
    count = [0]

    def cb(_):
        count[0] += 1

    maxiter = CG_ITER_FACTOR * n if maxiter is None else maxiter
    x, info = spla.cg(A, b, x0=x0, rtol=rtol, atol=atol, maxiter=maxiter, M=M, callback=cb)
    if info != 0:
        residual = float(np.linalg.norm(b - A @ x))
        raise SolverError(f"conjugate gradients stopped, residual {residual:.3e}", residual)
    return x, count[0]


def strain(jac):
    return 0.5 * (jac + np.swapaxes(jac, -1, -2))


def stress(eps, lame):
    lam, mu = lame
    d = eps.shape[-1]
    tr = np.trace(eps, axis1=-2, axis2=-1)
    return 2.0 * mu * eps + lam * tr[..., None, None] * np.eye(d)


def boundary_traction_vector(space, facet_ids, g):
    """Load vector of a constant traction g on the given boundary facets.

    2D restates ``boundary_vector_load`` (``fem.py:441-448``) with its
    2-point Gauss rule; for constant g each facet node receives
    g * |f| * (1 - x1 + 1 - x2)/2 resp. g * |f| * (x1 + x2)/2.  3D uses the
    exact P1 facet integral g |f| / 3 per vertex.
    """
    g = np.asarray(g, dtype=float)
    d = space.dim
    facets = space.grid.boundary_facets[facet_ids]
    meas = space.grid.facet_measures()[facet_ids]
    out = np.zeros(space.dof_count)
    if d == 2:
        gp = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
        basis = np.stack([1.0 - gp, gp], axis=1)  # (q, node)
        w = np.repeat((meas / 2.0)[:, None], 2, axis=1)
        elems = np.einsum("fqc,qa->fac", w[:, :, None] * np.broadcast_to(g, (len(facets), 2, 2)), basis)
    else:
        elems = np.broadcast_to((meas / 3.0)[:, None, None] * g[None, None, :], (len(facets), 3, 3))
    dofs = (d * facets[:, :, None] + np.arange(d)[None, None, :])
    np.add.at(out, dofs.reshape(len(facets), -1), elems.reshape(len(facets), -1))
    return out


def body_force_vector(space, f):
    """Exact P1 load of a constant body force (reference ``vector_load``, ``fem.py:419-425``)."""
    f = np.asarray(f, dtype=float)
    nq = space.quad_weights.shape[1]
    f_q = np.broadcast_to(f, space.quad_weights.shape + (space.dim,))
    elems = np.einsum("tqc,qa->tac", space.quad_weights[:, :, None] * f_q, space.bary)
    return space.assemble_vector(elems.reshape(len(elems), -1))


def clamp_dofs(space, facet_ids):
    """All dofs of the nodes on the given facets (``DirichletSet.on_tags``, ``fem.py:248-266``)."""
    nodes = np.unique(space.grid.boundary_facets[facet_ids])
    d = space.value_rank
    return (d * nodes[:, None] + np.arange(d)[None, :]).reshape(-1)

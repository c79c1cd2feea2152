"""Structured simplex meshes of boxes (oracle; test infrastructure only).

2D restates ``build_rect_mesh`` (reference ``mesh.py:113-170``): vertices from
``np.linspace`` with ``vid = j*(nx+1)+i`` (``mesh.py:132-138``); each cell
(i, j) yields a lower triangle (a, b, c) = (v(i,j), v(i+1,j), v(i+1,j+1)) at
row 2(j*nx+i) and an upper triangle (a, c, d) = (v(i,j), v(i+1,j+1),
v(i,j+1)) at the next row (``mesh.py:140-150``); boundary facets walk CCW:
bottom, right, top, left (``mesh.py:152-157``); tags come from midpoint
predicates, first match wins (``mesh.py:182-198``).

3D is new (the reference is 2D only, ``fem.py:63-64``): vertices
``vid = (k*(ny+1)+j)*(nx+1)+i``; cell c = (k*ny+j)*nx+i is split into the six
Kuhn tetrahedra t = 6c+m, m indexing the axis permutations
``KUHN_PERMS[m] = (a, b, c)``; tet m has the path vertices
v0, v0+e_a, v0+e_a+e_b, v0+e_a+e_b+e_c (local order = path order).  All six
share the cube diagonal v000-v111, so the split is conforming.  Boundary
facets are the triangles of the six faces (order x0, x1, y0, y1, z0, z1,
squares row-major in the two in-face axes, both triangles of a square split
along the in-face diagonal through the low/high corner, which is the trace
of the Kuhn split).
"""

import math

import numpy as np

KUHN_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))


class Grid:
    """Structured mesh of [lo, hi] with n cells per axis (d = 2 or 3)."""

    def __init__(self, lo, hi, n, tag_rules=None):
        self.dim = len(n)
        assert self.dim in (2, 3) and len(lo) == len(hi) == self.dim
        self.lo = tuple(float(v) for v in lo)
        self.hi = tuple(float(v) for v in hi)
        self.n = tuple(int(v) for v in n)
        axes = [np.linspace(self.lo[a], self.hi[a], self.n[a] + 1) for a in range(self.dim)]
        self.axes = axes
        if self.dim == 2:
            gx, gy = np.meshgrid(axes[0], axes[1])
            self.vertices = np.column_stack([gx.ravel(), gy.ravel()])
            self.elements = _rect_triangles(*self.n)
            self.boundary_facets = _rect_facets(*self.n)
        else:
            gz, gy, gx = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
            self.vertices = np.column_stack([gx.ravel(), gy.ravel(), gz.ravel()])
            self.elements = _kuhn_tets(*self.n)
            self.boundary_facets = _box_facets(*self.n)
        self.facet_tags = np.zeros(len(self.boundary_facets), dtype=np.int32)
        if tag_rules:
            self.facet_tags = tag_boundary(self, tag_rules)

    # -- sizes -----------------------------------------------------------------
    @property
    def num_vertices(self):
        return self.vertices.shape[0]

    @property
    def num_elements(self):
        return self.elements.shape[0]

    @property
    def measure(self):
        return float(np.prod([h - l for l, h in zip(self.lo, self.hi)]))

    @property
    def spacing(self):
        return tuple((h - l) / m for l, h, m in zip(self.lo, self.hi, self.n))

    # -- per-element geometry ------------------------------------------------------
    def element_measures(self):
        p = self.vertices[self.elements]
        edges = p[:, 1:] - p[:, :1]
        det = np.linalg.det(edges) if self.dim == 3 else (
            edges[:, 0, 0] * edges[:, 1, 1] - edges[:, 0, 1] * edges[:, 1, 0])
        return np.abs(det) / math.factorial(self.dim)

    def facet_midpoints(self):
        return self.vertices[self.boundary_facets].mean(axis=1)

    def facet_measures(self):
        p = self.vertices[self.boundary_facets]
        if self.dim == 2:
            return np.linalg.norm(p[:, 1] - p[:, 0], axis=1)
        return 0.5 * np.linalg.norm(np.cross(p[:, 1] - p[:, 0], p[:, 2] - p[:, 0]), axis=1)

    def facets_with_tag(self, tag):
        tags = np.atleast_1d(np.asarray(tag, dtype=np.int32))
        return np.nonzero(np.isin(self.facet_tags, tags))[0]


def _rect_triangles(nx, ny):
    vid = lambda i, j: j * (nx + 1) + i
    ii, jj = np.meshgrid(np.arange(nx), np.arange(ny))
    ii, jj = ii.ravel(), jj.ravel()
    a, b, c, d = vid(ii, jj), vid(ii + 1, jj), vid(ii + 1, jj + 1), vid(ii, jj + 1)
    tri = np.empty((2 * nx * ny, 3), dtype=np.int64)
    tri[0::2] = np.column_stack([a, b, c])
    tri[1::2] = np.column_stack([a, c, d])
    return tri


def _rect_facets(nx, ny):
    vid = lambda i, j: j * (nx + 1) + i
    walk = [(vid(i, 0), vid(i + 1, 0)) for i in range(nx)]
    walk += [(vid(nx, j), vid(nx, j + 1)) for j in range(ny)]
    walk += [(vid(i + 1, ny), vid(i, ny)) for i in range(nx - 1, -1, -1)]
    walk += [(vid(0, j + 1), vid(0, j)) for j in range(ny - 1, -1, -1)]
    return np.array(walk, dtype=np.int64)


def _kuhn_tets(nx, ny, nz):
    vid = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i
    kk, jj, ii = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    ii, jj, kk = ii.ravel(), jj.ravel(), kk.ravel()
    tets = np.empty((6 * nx * ny * nz, 4), dtype=np.int64)
    for m, perm in enumerate(KUHN_PERMS):
        off = np.zeros(3, dtype=np.int64)
        cols = [vid(ii, jj, kk)]
        for axis in perm:
            off[axis] += 1
            cols.append(vid(ii + off[0], jj + off[1], kk + off[2]))
        tets[m::6] = np.column_stack(cols)
    return tets


def _box_facets(nx, ny, nz):
    vid = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i
    out = []
    n = (nx, ny, nz)
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        for side in (0, n[axis]):
            for q in range(n[v]):
                for p in range(n[u]):
                    def node(du, dv):
                        idx = [0, 0, 0]
                        idx[axis] = side
                        idx[u] = p + du
                        idx[v] = q + dv
                        return vid(*idx)
                    out.append((node(0, 0), node(1, 0), node(1, 1)))
                    out.append((node(0, 0), node(1, 1), node(0, 1)))
    return np.array(out, dtype=np.int64)


def tag_boundary(grid, rules):
    """First-match midpoint tagging (reference ``mesh.py:182-198``)."""
    mids = grid.facet_midpoints()
    tags = np.zeros(len(mids), dtype=np.int32)
    unset = np.ones(len(mids), dtype=bool)
    for tag, predicate in rules:
        assert tag != 0
        hit = np.asarray(predicate(mids), dtype=bool) & unset
        tags[hit] = tag
        unset &= ~hit
    return tags


def mesh_diameter(grid):
    """Squared nominal element size (reference ``mesh.py:173-179`` in 2D;
    ``PAPER.md:958-966`` in 3D): 4|D|/(N_T sqrt 3), resp. (6 sqrt2 |D|/N_T)^(2/3)."""
    if grid.dim == 2:
        return 4.0 * grid.measure / (grid.num_elements * np.sqrt(3.0))
    return (6.0 * np.sqrt(2.0) * grid.measure / grid.num_elements) ** (2.0 / 3.0)


def level_set_h(grid):
    """Interface length scale h = sqrt(mesh_diameter) (reference ``levelset.py:51``)."""
    return math.sqrt(mesh_diameter(grid))

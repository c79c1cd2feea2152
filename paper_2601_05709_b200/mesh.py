"""Structured simplex meshes of boxes (drop-in for reference ``mesh.py``).

``build_rect_mesh`` keeps the reference's signature and numbering
(``mesh.py:113-170``): vertices ``vid = j*(nx+1)+i`` on ``np.linspace``
coordinates, lower/upper triangles per cell, boundary facets walked CCW
(bottom, right, top, left), first-match midpoint tags (``mesh.py:182-198``).
``build_box_mesh`` is the 3D extension (six Kuhn tetrahedra per cell).

Only the boundary facets (and their tags) live on the host -- they are what
the boundary-condition and load APIs consume.  The device never needs
connectivity: every kernel indexes the structured lattice in closed form.
``vertices`` / ``triangles`` (``elements``) are produced on demand by the
device kernels ``lsg_mesh_vertices`` / ``lsg_mesh_elements`` and copied to the
host, bit-identical to the reference's arrays.
"""

import math
from functools import cached_property

import numpy as np
import torch

from . import _lib
from .errors import ConfigError

__all__ = ["StructuredMesh", "RectMesh", "BoxMesh", "build_rect_mesh", "build_box_mesh",
           "mesh_diameter", "tag_boundary"]


class StructuredMesh:
    """Mesh of the box [lo, hi] with n cells per axis (dim 2 or 3)."""

    def __init__(self, lo, hi, n, facet_tags=None):
        self.dim = len(n)
        self.lo = tuple(float(v) for v in lo)
        self.hi = tuple(float(v) for v in hi)
        self.n = tuple(int(v) for v in n)
        self.grid = _lib.make_grid(self.dim, self.n, self.lo, self.hi)
        self.boundary_facets = _box_facets(self.n) if self.dim == 3 else _rect_facets(*self.n)
        if facet_tags is None:
            facet_tags = np.zeros(len(self.boundary_facets), dtype=np.int32)
        self.facet_tags = np.asarray(facet_tags, dtype=np.int32)
        # device workspaces / scratch buffers of solves on this mesh (fem._workspace,
        # levelset._Scratch): they live and die with the mesh object
        self.device_cache = {}

    # -- sizes --------------------------------------------------------------------
    @property
    def num_vertices(self):
        return int(np.prod([m + 1 for m in self.n]))

    @property
    def num_elements(self):
        cells = int(np.prod(self.n))
        return 2 * cells if self.dim == 2 else 6 * cells

    @property
    def measure(self):
        return float(np.prod([h - l for l, h in zip(self.lo, self.hi)]))

    area = measure  # reference RectMesh.area (mesh.py:58-61)

    @property
    def spacing(self):
        return tuple((h - l) / m for l, h, m in zip(self.lo, self.hi, self.n))

    @property
    def bounds(self):
        if self.dim == 2:
            return (self.lo[0], self.lo[1], self.hi[0], self.hi[1])
        return self.lo + self.hi

    # -- host-side coordinates (linspace, bit-identical to the reference) -----------
    @cached_property
    def axes(self):
        return [np.linspace(self.lo[a], self.hi[a], self.n[a] + 1) for a in range(self.dim)]

    def node_coords(self, nodes):
        """Coordinates of the given node ids, (m, dim)."""
        nodes = np.asarray(nodes, dtype=np.int64)
        out = np.empty((len(nodes), self.dim))
        rest = nodes
        for a in range(self.dim):
            m = self.n[a] + 1
            out[:, a] = self.axes[a][rest % m]
            rest = rest // m
        return out

    @cached_property
    def facet_midpoints(self):
        pts = self.node_coords(self.boundary_facets.reshape(-1)).reshape(
            self.boundary_facets.shape + (self.dim,))
        return pts.mean(axis=1)

    @cached_property
    def facet_measures(self):
        pts = self.node_coords(self.boundary_facets.reshape(-1)).reshape(
            self.boundary_facets.shape + (self.dim,))
        if self.dim == 2:
            return np.linalg.norm(pts[:, 1] - pts[:, 0], axis=1)
        return 0.5 * np.linalg.norm(np.cross(pts[:, 1] - pts[:, 0], pts[:, 2] - pts[:, 0]), axis=1)

    @property
    def facet_lengths(self):
        return self.facet_measures

    def facets_with_tag(self, tag):
        tags = np.atleast_1d(np.asarray(tag, dtype=np.int32))
        return np.nonzero(np.isin(self.facet_tags, tags))[0]

    def with_tags(self, facet_tags):
        return type(self)._rebuild(self, facet_tags)

    @classmethod
    def _rebuild(cls, mesh, facet_tags):
        out = cls.__new__(cls)
        out.__dict__.update({k: v for k, v in mesh.__dict__.items()
                             if k not in ("facet_midpoints", "facet_measures")})
        out.facet_tags = np.asarray(facet_tags, dtype=np.int32)
        return out

    # -- device-generated full arrays -------------------------------------------------
    def device_vertices(self):
        out = torch.empty((self.num_vertices, self.dim), dtype=torch.float64, device="cuda")
        _lib.call("lsg_mesh_vertices", self.grid, _lib.ptr(out), _lib.stream())
        return out

    def device_elements(self):
        out = torch.empty((self.num_elements, self.dim + 1), dtype=torch.int32, device="cuda")
        _lib.call("lsg_mesh_elements", self.grid, _lib.ptr(out), _lib.stream())
        return out

    @cached_property
    def vertices(self):
        return self.device_vertices().cpu().numpy()

    @cached_property
    def elements(self):
        return self.device_elements().cpu().numpy()


class RectMesh(StructuredMesh):
    """2D structured triangle mesh (reference ``RectMesh``, ``mesh.py:25-110``)."""

    @property
    def nx(self):
        return self.n[0]

    @property
    def ny(self):
        return self.n[1]

    @property
    def num_triangles(self):
        return self.num_elements

    @property
    def triangles(self):
        return self.elements


class BoxMesh(StructuredMesh):
    """3D structured Kuhn-tetrahedron mesh."""

    @property
    def tetrahedra(self):
        return self.elements


def build_rect_mesh(bounds, nx, ny, tag_rules=None):
    """Triangulate ``bounds = (x0, y0, x1, y1)`` with an nx by ny grid (``mesh.py:113-170``)."""
    if not (isinstance(nx, (int, np.integer)) and isinstance(ny, (int, np.integer))):
        raise ConfigError(f"cell counts must be integers, got nx={nx!r} ny={ny!r}")
    if nx < 1 or ny < 1:
        raise ConfigError(f"cell counts must be >= 1, got nx={nx} ny={ny}")
    x0, y0, x1, y1 = map(float, bounds)
    if not (x1 > x0 and y1 > y0):
        raise ConfigError(f"bounds must satisfy x1 > x0 and y1 > y0, got {bounds}")
    mesh = RectMesh((x0, y0), (x1, y1), (int(nx), int(ny)))
    if tag_rules:
        mesh.facet_tags = tag_boundary(mesh, tag_rules)
    return mesh


def build_box_mesh(bounds, n, tag_rules=None):
    """Kuhn-tetrahedron mesh of ``bounds = (x0, y0, z0, x1, y1, z1)`` with n = (nx, ny, nz)."""
    if len(bounds) != 6 or len(n) != 3:
        raise ConfigError("box mesh needs 6 bounds and 3 cell counts")
    if any(not isinstance(m, (int, np.integer)) or m < 1 for m in n):
        raise ConfigError(f"cell counts must be integers >= 1, got {n}")
    lo, hi = tuple(map(float, bounds[:3])), tuple(map(float, bounds[3:]))
    if not all(h > l for l, h in zip(lo, hi)):
        raise ConfigError(f"bounds must satisfy hi > lo, got {bounds}")
    mesh = BoxMesh(lo, hi, tuple(int(m) for m in n))
    if tag_rules:
        mesh.facet_tags = tag_boundary(mesh, tag_rules)
    return mesh


def mesh_diameter(mesh):
    """Squared nominal element size: 4|D|/(N_T sqrt 3) in 2D (``mesh.py:173-179``),
    (6 sqrt2 |D| / N_T)^(2/3) in 3D (``PAPER.md:958-966``)."""
    if mesh.dim == 2:
        return 4.0 * mesh.measure / (mesh.num_elements * np.sqrt(3.0))
    return (6.0 * np.sqrt(2.0) * mesh.measure / mesh.num_elements) ** (2.0 / 3.0)


def tag_boundary(mesh, rules):
    """First-match midpoint tagging (``mesh.py:182-198``)."""
    mids = mesh.facet_midpoints
    tags = np.zeros(len(mids), dtype=np.int32)
    unset = np.ones(len(mids), dtype=bool)
    for tag, predicate in rules:
        if tag == 0:
            raise ConfigError("tag 0 is reserved for untagged facets")
        hit = np.asarray(predicate(mids), dtype=bool) & unset
        tags[hit] = tag
        unset &= ~hit
    return tags


def _rect_facets(nx, ny):
    i = np.arange(nx)
    j = np.arange(ny)
    vid = lambda a, b: b * (nx + 1) + a
    bottom = np.stack([vid(i, 0), vid(i + 1, 0)], axis=1)
    right = np.stack([vid(nx, j), vid(nx, j + 1)], axis=1)
    ir = i[::-1]
    top = np.stack([vid(ir + 1, ny), vid(ir, ny)], axis=1)
    jr = j[::-1]
    left = np.stack([vid(0, jr + 1), vid(0, jr)], axis=1)
    return np.concatenate([bottom, right, top, left]).astype(np.int64)


def _box_facets(n):
    nx, ny, nz = n
    vid = lambda i, j, k: (k * (ny + 1) + j) * (nx + 1) + i
    out = []
    for axis in range(3):
        u, v = [a for a in range(3) if a != axis]
        pu, qv = np.meshgrid(np.arange(n[u]), np.arange(n[v]))
        pu, qv = pu.ravel(), qv.ravel()
        for side in (0, n[axis]):
            def node(du, dv):
                idx = [None, None, None]
                idx[axis] = np.full_like(pu, side)
                idx[u] = pu + du
                idx[v] = qv + dv
                return vid(*idx)
            a, b, c, d = node(0, 0), node(1, 0), node(1, 1), node(0, 1)
            tri = np.empty((2 * len(pu), 3), dtype=np.int64)
            tri[0::2] = np.stack([a, b, c], axis=1)
            tri[1::2] = np.stack([a, c, d], axis=1)
            out.append(tri)
    return np.concatenate(out)

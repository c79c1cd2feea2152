"""Level-set fields and the explicit level-set update (drop-in for reference ``levelset.py``).

``transport`` and ``reinitialize`` keep the reference's signatures, argument
checks and "returns a new field, input untouched" semantics
(``levelset.py:137-216``), but integrate the north star's explicit scheme on
the device (``csrc/levelset.cu``; statement and CPU oracle in
``oracle/levelset.py``):

* transport: phi_t + theta . grad phi = [smooth] h^2 lap phi by conservative
  face-velocity upwinding, forward Euler, nsub = max(steps,
  ceil(t_end (speed + kappa) / CFL)) substeps, CFL = 1/2;
* reinitialize: phi_t = -S (|grad phi| - 1) + h^2 lap phi (Godunov), frozen
  S = phi0 / sqrt(phi0^2 + h^2), nsub = max(iters, ceil(t_final (sum 1/h_d +
  kappa) / CFL)).
"""

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import ConfigError, SolverError
from .fem import FemField, FunctionSpace, to_device
from .mesh import mesh_diameter

__all__ = ["LevelSetField", "InitialLevelSpec", "initial_level", "transport", "reinitialize",
           "transport_substeps", "reinit_substeps", "cfl_speed", "CFL"]

CFL = 0.5


class LevelSetField:
    """Scalar P1 field whose subzero set is the working domain (``levelset.py:33-67``)."""

    def __init__(self, field, h):
        self.field = field
        self.h = float(h)

    @classmethod
    def from_field(cls, fem_field):
        if not bool(torch.isfinite(fem_field.values).all()):
            raise ConfigError("level-set field has non-finite nodal values")
        return cls(fem_field, math.sqrt(mesh_diameter(fem_field.space.mesh)))

    @property
    def values(self):
        return self.field.values

    @property
    def space(self):
        return self.field.space

    @property
    def mesh(self):
        return self.field.space.mesh

    def indicator_quad(self):
        """Quadrature-point indicator of the subzero region, (E, nq) on the device."""
        mesh = self.mesh
        nq = 3 if mesh.dim == 2 else 4
        chi = torch.empty((mesh.num_elements, nq), dtype=torch.float64, device="cuda")
        _lib.call("lsg_indicator_quad", mesh.grid, _lib.ptr(self.values), _lib.ptr(chi),
                  _lib.stream())
        return chi


@dataclass(frozen=True)
class InitialLevelSpec:
    """Union-of-balls initializer phi = factor * max_k (r_k - |x - c_k|) (``levelset.py:70-95``)."""

    centers: tuple
    radii: tuple
    factor: float = 1.0
    ord: float = 2

    def __post_init__(self):
        if len(self.centers) != len(self.radii) or len(self.radii) < 1:
            raise ConfigError("need matching nonempty centers/radii")
        if any(r <= 0.0 for r in self.radii):
            raise ConfigError("ball radii must be positive")
        if self.factor == 0.0:
            raise ConfigError("initial level factor must be nonzero")
        if self.ord not in (2, math.inf):
            raise ConfigError(f"norm order must be 2 or inf, got {self.ord}")


def initial_level(spec, space):
    if space.value_rank != 1:
        raise ConfigError("initial level set needs a scalar space")
    pts = space.mesh.device_vertices()
    best = torch.full((pts.shape[0],), -math.inf, dtype=torch.float64, device="cuda")
    for center, radius in zip(spec.centers, spec.radii):
        diff = pts - torch.as_tensor(center, dtype=torch.float64, device="cuda")
        dist = torch.linalg.vector_norm(diff, ord=spec.ord, dim=1)
        best = torch.maximum(best, radius - dist)
    return LevelSetField.from_field(FemField(space, spec.factor * best))


class _Scratch:
    """Per-mesh device scratch buffers, cached on the mesh object (freed with it)."""

    def get(self, mesh, name, numel, dtype=torch.float64):
        key = ("scratch", name, numel, dtype)
        t = mesh.device_cache.get(key)
        if t is None:
            t = torch.empty(numel, dtype=dtype, device="cuda")
            mesh.device_cache[key] = t
        return t


_SCRATCH = _Scratch()


def cfl_speed(theta):
    """max_i sum_d |theta_d,i| / h_d, computed on the device (one host read)."""
    cached = getattr(theta, "_cfl_speed", None)
    if cached is not None:
        return cached
    mesh = theta.space.mesh
    out = _SCRATCH.get(mesh, "cfl_out", 1)
    part = _SCRATCH.get(mesh, "cfl_part", 4096)
    cnt = _SCRATCH.get(mesh, "cfl_cnt", 1, torch.int32)
    if not getattr(cnt, "_armed", False):
        cnt.zero_()
        cnt._armed = True
    _lib.call("lsg_cfl_speed", mesh.grid, _lib.ptr(theta.values), _lib.ptr(out), _lib.ptr(part),
              _lib.ptr(cnt), _lib.stream())
    return float(out.item())


def transport_substeps(mesh, speed, t_end, steps, smooth, h):
    kappa = h * h * sum(2.0 / (s * s) for s in mesh.spacing) if smooth else 0.0
    return max(int(steps), int(math.ceil(t_end * (speed + kappa) / CFL)))


def reinit_substeps(mesh, iters, t_final, h):
    speed = sum(1.0 / s for s in mesh.spacing)
    kappa = h * h * sum(2.0 / (s * s) for s in mesh.spacing)
    return max(int(iters), int(math.ceil(t_final * (speed + kappa) / CFL)))


def _check_velocity_field(phi, theta):
    if theta.space.value_rank != phi.mesh.dim:
        raise ConfigError("transport velocity must live on a vector space")
    if theta.space.mesh is not phi.space.mesh:
        raise ConfigError("velocity and level set use different meshes")


PG_RTOL = 1e-14  # BiCGStab tolerance of the reference scheme's step solves (reference: SuperLU)


BICG_LOG = None  # set to a list to record (iterations, relative residual) per solve


def _bicgstab(op, b, x, mesh):
    work = _SCRATCH.get(mesh, "bicg_work", int(_lib.load().lsg_bicgstab_work_doubles(mesh.grid)))
    iters = ctypes.c_int32(0)
    resid = ctypes.c_double(0.0)
    try:
        _lib.call("lsg_bicgstab", op, _lib.ptr(b), _lib.ptr(x), _lib.ptr(work), PG_RTOL, 4000,
                  ctypes.byref(iters), ctypes.byref(resid), _lib.stream())
    except SolverError as exc:
        raise SolverError(str(exc), residual=float(resid.value)) from None
    if BICG_LOG is not None:
        BICG_LOG.append((int(iters.value), float(resid.value)))
    return int(iters.value)


def _transport_pg(phi, theta, t_end, steps, smooth):
    """Crank-Nicolson Petrov-Galerkin transport (``levelset.py:137-169``) on the device."""
    mesh = phi.mesh
    if mesh.dim != 2:
        raise ConfigError("the reference (pg) level-set scheme is 2D only")
    dt = t_end / steps
    th = theta.values
    lhs = _lib.make_op(_lib.LSG_OP_PG_TRANSPORT, mesh.grid, None, (dt, phi.h, 1.0, float(smooth)), (th,))
    rhs = _lib.make_op(_lib.LSG_OP_PG_TRANSPORT, mesh.grid, None, (dt, phi.h, -1.0, float(smooth)), (th,))
    vals = phi.values.clone()
    b = torch.empty_like(vals)
    for _ in range(steps):
        _lib.call("lsg_apply", rhs, 1, _lib.ptr(vals), _lib.ptr(b), _lib.stream())
        _bicgstab(lhs, b, vals, mesh)
    out = LevelSetField(FemField(phi.space, vals), phi.h)
    out.substeps = steps
    return out


def _reinitialize_pg(phi, iters, t_final):
    """Petrov-Galerkin Euler/AB2 reinitialisation (``levelset.py:172-216``) on the device."""
    mesh = phi.mesh
    if mesh.dim != 2:
        raise ConfigError("the reference (pg) level-set scheme is 2D only")
    dt = t_final / iters
    phi0 = phi.values
    cur, prev = phi0.clone(), phi0.clone()  # duplicated history: step one is Euler
    b = torch.empty_like(cur)
    for _ in range(iters):
        op = _lib.make_op(_lib.LSG_OP_PG_REINIT, mesh.grid, None, (dt, phi.h), (phi0, cur, prev))
        _lib.call("lsg_pg_reinit_rhs", op, _lib.ptr(b), _lib.stream())
        x = cur.clone()
        _bicgstab(op, b, x, mesh)
        prev, cur = cur, x
    out = LevelSetField(FemField(phi.space, cur), phi.h)
    out.substeps = iters
    return out


def transport(phi, theta, t_end, steps, smooth=False, scheme="explicit"):
    """Advect phi along theta for time t_end (``levelset.py:137-169`` signature).

    ``scheme="explicit"`` (default): the north star's explicit upwind HJ
    step under CFL; ``scheme="pg"``: the reference's own Crank-Nicolson
    Petrov-Galerkin step (2D).
    """
    if t_end <= 0.0:
        raise ConfigError(f"transport needs t_end > 0, got {t_end}")
    if steps < 1:
        raise ConfigError(f"transport needs steps >= 1, got {steps}")
    _check_velocity_field(phi, theta)
    if scheme == "pg":
        return _transport_pg(phi, theta, t_end, steps, smooth)
    if scheme != "explicit":
        raise ConfigError(f"unknown level-set scheme {scheme!r}")
    mesh = phi.mesh
    nsub = transport_substeps(mesh, cfl_speed(theta), t_end, steps, smooth, phi.h)
    n = mesh.num_vertices
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    tmp = _SCRATCH.get(mesh, "ls_tmp", n)
    _lib.call("lsg_transport", mesh.grid, _lib.ptr(phi.values), _lib.ptr(theta.values),
              float(t_end / nsub), int(nsub), int(bool(smooth)), float(phi.h), _lib.ptr(out),
              _lib.ptr(tmp), _lib.stream())
    res = LevelSetField(FemField(phi.space, out), phi.h)
    res.substeps = nsub
    return res


def reinitialize(phi, iters, t_final, scheme="explicit"):
    """Drive phi toward the signed distance of its zero set (``levelset.py:172-216`` signature)."""
    if iters < 2:
        raise ConfigError(f"reinitialization needs iters >= 2, got {iters}")
    if t_final <= 0.0:
        raise ConfigError(f"reinitialization needs t_final > 0, got {t_final}")
    if scheme == "pg":
        return _reinitialize_pg(phi, iters, t_final)
    if scheme != "explicit":
        raise ConfigError(f"unknown level-set scheme {scheme!r}")
    mesh = phi.mesh
    nsub = reinit_substeps(mesh, iters, t_final, phi.h)
    n = mesh.num_vertices
    out = torch.empty(n, dtype=torch.float64, device="cuda")
    tmp = _SCRATCH.get(mesh, "ls_tmp", n)
    sgn = _SCRATCH.get(mesh, "ls_sgn", n)
    _lib.call("lsg_reinit", mesh.grid, _lib.ptr(phi.values), float(t_final / nsub), int(nsub),
              float(phi.h), _lib.ptr(out), _lib.ptr(tmp), _lib.ptr(sgn), _lib.stream())
    res = LevelSetField(FemField(phi.space, out), phi.h)
    res.substeps = nsub
    return res

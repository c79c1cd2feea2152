"""The five BASELINE.json configurations as plain data.

Each ``Case`` pins what the BASELINE text leaves open, exactly as SURVEY
Appendix B recommends:

* Lame pair from E = 1, nu = 0.3: plane stress in 2D, standard in 3D;
* ersatz 1e-3; H1 velocity form (mass 1, alpha = 1e-2);
* volume target = fraction * |D|; exactly ``niter`` iterations
  (``start_to_check = niter``); reinit every 5 iterations, (8, 0.1);
* cfg2 loads: traction density magnitude m_k (downward) on top-edge facets
  whose midpoint lies within 0.01 of x_k = 0.5 + 3k/7 (0.02-wide patch),
  m = default_rng(0).uniform(0.5, 1.5, 8); supports: bottom facets with
  midpoint x < 0.02 or x > 3.98;
* cfg3/cfg5 load patch: x = 2 face triangles whose centroid satisfies
  |y - 0.5| < 0.1 and |z - 0.5| < 0.1;
* cfg4: phi is a Gaussian random field (white noise from
  default_rng(0).standard_normal on the node lattice, Gaussian filter of
  correlation length 0.05 applied in Fourier space, standardised); bottom
  edge clamped; body force (0, -1).

``scale`` divides every cell count (parity tests run the same geometry on
coarser grids).  Used by the product harness (bench.py) and by the tests,
which hand the same data to the CPU oracle.
"""

import math
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

__all__ = ["Case", "case", "CASES", "gaussian_random_field"]


@dataclass(frozen=True)
class Case:
    name: str
    lo: tuple
    hi: tuple
    n: tuple
    E: float = 1.0
    nu: float = 0.3
    ersatz: float = 1e-3
    fixed: Callable = None                 # predicate on facet midpoints
    loads: tuple = ()                      # ((traction, predicate), ...)
    body_force: Optional[tuple] = None
    volume_fraction: float = 0.5
    phi0: Callable = None                  # points (N, d) -> (N,)
    niter: int = 50
    reinit_step: Optional[int] = 5
    reinit_pars: tuple = (8, 0.1)
    h1: tuple = (1.0, 1e-2)

    @property
    def dim(self):
        return len(self.n)

    @property
    def measure(self):
        return float(np.prod([h - l for l, h in zip(self.lo, self.hi)]))

    @property
    def volume(self):
        return self.volume_fraction * self.measure

    @property
    def lame(self):
        E, nu = self.E, self.nu
        if self.dim == 2:
            return (E * nu / (1.0 - nu * nu), E / (2.0 * (1.0 + nu)))
        return (E * nu / ((1.0 + nu) * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu)))

    @property
    def num_nodes(self):
        return int(np.prod([m + 1 for m in self.n]))


def gaussian_random_field(shape, spacing, corr, seed=0):
    """Standardised FFT-filtered white noise on a node lattice (cfg4 phi)."""
    rng = np.random.default_rng(seed)
    noise = rng.standard_normal(shape)
    spec = np.fft.rfftn(noise)
    freqs = [np.fft.fftfreq(m, d=h) for m, h in zip(shape[:-1], spacing[:-1])]
    freqs.append(np.fft.rfftfreq(shape[-1], d=spacing[-1]))
    grids = np.meshgrid(*freqs, indexing="ij")
    k2 = sum((2.0 * math.pi * f) ** 2 for f in grids)
    spec *= np.exp(-0.5 * k2 * corr * corr)
    out = np.fft.irfftn(spec, s=shape, axes=tuple(range(len(shape))))
    out -= out.mean()
    out /= out.std()
    return out


def _cfg1(scale=1):
    nx, ny = 160 // scale, 80 // scale
    return Case(
        name="cfg1", lo=(0.0, 0.0), hi=(2.0, 1.0), n=(nx, ny),
        fixed=lambda p: p[:, 0] < 1e-12,
        loads=(((0.0, -1.0), lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55)),),
        volume_fraction=0.5,
        phi0=lambda p: -np.cos(6 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) - 0.4,
        niter=50)


CFG2_MAGNITUDES = tuple(np.random.default_rng(0).uniform(0.5, 1.5, 8).tolist())


def _cfg2(scale=1):
    nx, ny = 1024 // scale, 256 // scale
    xs = [0.5 + 3.0 * k / 7.0 for k in range(8)]
    half = max(0.01, 0.5 * 4.0 / nx + 1e-9)  # at least one facet on coarse grids

    def patch(xk):
        return lambda p: (p[:, 1] > 1.0 - 1e-12) & (np.abs(p[:, 0] - xk) < half)

    loads = tuple(((0.0, -m), patch(x)) for x, m in zip(xs, CFG2_MAGNITUDES))
    strip = max(0.02, 4.0 / nx + 1e-9)
    return Case(
        name="cfg2", lo=(0.0, 0.0), hi=(4.0, 1.0), n=(nx, ny),
        fixed=lambda p: (p[:, 1] < 1e-12) & ((p[:, 0] < strip) | (p[:, 0] > 4.0 - strip)),
        loads=loads, volume_fraction=0.4,
        phi0=lambda p: -np.cos(8 * np.pi * p[:, 0] / 4.0) * np.cos(4 * np.pi * p[:, 1]) - 0.3,
        niter=40)


def _face_patch(x, ny):
    # |y - 0.5| < 0.1, |z - 0.5| < 0.1 (widened on coarse test grids so that the
    # patch always contains facets)
    half = max(0.1, 0.75 / ny)
    return lambda p: (p[:, 0] > x - 1e-12) & (np.abs(p[:, 1] - 0.5) < half) & (np.abs(p[:, 2] - 0.5) < half)


def _cfg3(scale=1):
    n = (96 // scale, 48 // scale, 48 // scale)
    return Case(
        name="cfg3", lo=(0.0, 0.0, 0.0), hi=(2.0, 1.0, 1.0), n=n,
        fixed=lambda p: p[:, 0] < 1e-12,
        loads=(((0.0, -1.0, 0.0), _face_patch(2.0, n[1])),),
        volume_fraction=0.3,
        phi0=lambda p: -np.cos(4 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) * np.cos(4 * np.pi * p[:, 2]) - 0.3,
        niter=30)


def _cfg4(scale=1):
    nx, ny = 4096 // scale, 2048 // scale

    def phi0(p, nx=nx, ny=ny):
        f = gaussian_random_field((ny + 1, nx + 1), (1.0 / ny, 2.0 / nx), 0.05, seed=0)
        return f.reshape(-1)

    return Case(
        name="cfg4", lo=(0.0, 0.0), hi=(2.0, 1.0), n=(nx, ny),
        fixed=lambda p: p[:, 1] < 1e-12, loads=(), body_force=(0.0, -1.0),
        volume_fraction=0.5, phi0=phi0, niter=1, reinit_step=None)


def _cfg5(scale=1):
    n = (192 // scale, 96 // scale, 96 // scale)
    dirs = ((0.0, -1.0, 0.0), (0.0, 0.0, -1.0), (0.0, 1.0, 0.0), (0.0, 0.0, 1.0))
    patch = _face_patch(2.0, n[1])  # one patch (one facet tag) shared by the 4 load cases
    return Case(
        name="cfg5", lo=(0.0, 0.0, 0.0), hi=(2.0, 1.0, 1.0), n=n,
        fixed=lambda p: p[:, 0] < 1e-12,
        loads=tuple((d, patch) for d in dirs),
        volume_fraction=0.25,
        phi0=lambda p: -np.cos(6 * np.pi * p[:, 0]) * np.cos(6 * np.pi * p[:, 1]) * np.cos(6 * np.pi * p[:, 2]) - 0.3,
        niter=20)


CASES = {"cfg1": _cfg1, "cfg2": _cfg2, "cfg3": _cfg3, "cfg4": _cfg4, "cfg5": _cfg5}


def case(name, scale=1):
    return CASES[name](scale)


def load_tag_rules(c):
    """Boundary tag rules (tag 1 = clamp, then one tag per distinct load patch)
    and the tag of each load case; load cases sharing a patch predicate share
    its tag, since tagging is first-match-wins (mesh.py:182-198)."""
    rules, tags, seen = [(1, c.fixed)], [], {}
    for _, pred in c.loads:
        if id(pred) not in seen:
            seen[id(pred)] = 2 + len(seen)
            rules.append((seen[id(pred)], pred))
        tags.append(seen[id(pred)])
    return rules, tags


def build(c, device_phi=True):
    """Product-side model, initial level set and RunParams for a Case."""
    from . import (ComplianceModel, CompliancePlusModel, FemField, FunctionSpace, LevelSetField,
                   RunParams, build_box_mesh, build_rect_mesh)
    from .velocity import BilinearSpec

    rules, load_tags = load_tag_rules(c)
    if c.dim == 2:
        mesh = build_rect_mesh((c.lo[0], c.lo[1], c.hi[0], c.hi[1]), c.n[0], c.n[1], rules)
    else:
        mesh = build_box_mesh(c.lo + c.hi, c.n, rules)
    bil = BilinearSpec(mass_weight=c.h1[0], stiffness_weight=c.h1[1])
    kw = dict(lame=c.lame, bilinear=bil, ersatz=c.ersatz)
    if len(c.loads) > 1:
        model = CompliancePlusModel(mesh, 1, [(g, t) for (g, _), t in zip(c.loads, load_tags)],
                                    c.volume, **kw)
    elif len(c.loads) == 1:
        model = ComplianceModel(mesh, 1, load_tags[0], c.loads[0][0], c.volume, **kw)
    else:
        model = ComplianceModel(mesh, 1, None, None, c.volume, body_force=c.body_force, **kw)
    phi_vals = c.phi0(mesh.vertices if c.name != "cfg4" else None)
    phi = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), phi_vals))
    params = RunParams(niter=c.niter, start_to_check=c.niter, reinit_step=c.reinit_step,
                       reinit_pars=c.reinit_pars)
    return mesh, model, phi, params

"""Explicit level-set update (oracle; test infrastructure only).

The north star replaces the reference's Crank-Nicolson Petrov-Galerkin
transport (``levelset.py:137-169``) and Petrov-Galerkin AB2 reinitialisation
(``levelset.py:172-216``) by an explicit upwind Hamilton-Jacobi step under
CFL followed by an explicit reinitialisation.  This module is the CPU
statement of that scheme; the CUDA kernels must agree with it to 1e-10
relative L2.  It keeps the reference's conventions:

* nodal P1 phi on the structured node lattice; h = sqrt(mesh_diameter)
  (``levelset.py:51``);
* transport solves phi_t + theta . grad phi = [smooth] h^2 lap phi over
  (0, t_end] with at least ``steps`` substeps (``levelset.py:137-149``);
  homogeneous Neumann / no-inflow boundary (``levelset.py:141-143``,
  ``PAPER.md:992-996``): one-sided differences that would reach outside the
  box are zero, the Laplacian mirrors across the boundary;
* reinitialisation solves phi_t = -S (|grad phi| - 1) + h^2 lap phi with the
  frozen smoothed sign S = phi0 / sqrt(phi0^2 + h^2) (``levelset.py:175-188``)
  over (0, t_final] with at least ``iters`` substeps;
* space: first-order face-velocity upwind in conservative (lumped-P1) form
  for transport -- the plain nodal upwind form drifts the mass of phi by
  ~60 %/time on the reference's swirl test (``test_levelset.py:195-214``),
  this form conserves it to round-off -- and first-order Godunov for reinit;
  time: forward Euler; substep count
  nsub = max(steps, ceil(t * (speed + kappa) / CFL)), CFL = 1/2, where speed
  = max_i sum_d |v_d,i| / h_d (transport) or sum_d 1/h_d (reinit) and
  kappa = h^2 sum_d 2/h_d^2 when diffusion is on.
"""

import math

import numpy as np

CFL = 0.5


def _shape(grid):
    return tuple(m + 1 for m in reversed(grid.n))  # (nz,) ny, nx node lattice


def _diffs(f, axis, h):
    """Backward and forward differences along ``axis``; zero at the box faces."""
    dm = np.zeros_like(f)
    dp = np.zeros_like(f)
    sl = [slice(None)] * f.ndim
    lo = list(sl); hi = list(sl)
    lo[axis] = slice(1, None)
    hi[axis] = slice(None, -1)
    diff = (f[tuple(lo)] - f[tuple(hi)]) / h
    dm[tuple(lo)] = diff
    dp[tuple(hi)] = diff
    return dm, dp


def _laplacian(f, spacing):
    out = np.zeros_like(f)
    nd = f.ndim
    for k in range(nd):
        axis = nd - 1 - k  # lattice axis of spatial direction k
        h = spacing[k]
        pad = np.concatenate([np.take(f, [1], axis=axis), f, np.take(f, [-2], axis=axis)], axis=axis)
        n = f.shape[axis]
        left = np.take(pad, np.arange(0, n), axis=axis)
        right = np.take(pad, np.arange(2, n + 2), axis=axis)
        out += (left - 2.0 * f + right) / (h * h)
    return out


def transport_substeps(grid, theta, t_end, steps, smooth, h):
    spacing = grid.spacing
    d = grid.dim
    th = np.asarray(theta).reshape(-1, d)
    speed = float(np.max(sum(np.abs(th[:, k]) / spacing[k] for k in range(d))))
    kappa = h * h * sum(2.0 / (s * s) for s in spacing) if smooth else 0.0
    return max(int(steps), int(math.ceil(t_end * (speed + kappa) / CFL))), speed


def _face_upwind(f, th, spacing):
    """-(theta . grad phi) by face-velocity upwinding, lumped-P1 consistent.

    Along axis k the face between nodes i and i+1 carries the mean velocity
    V = (theta_i + theta_{i+1})/2 and the difference D = (phi_{i+1}-phi_i)/h;
    node i receives -min(V,0) D and node i+1 receives -max(V,0) D.  Faces
    outside the box do not exist (no inflow, zero flux) and the two boundary
    nodes of each line count twice, because their lumped P1 mass is h/2.
    Summed with the lumped weights the scheme changes the mass of phi only by
    the discrete integral of phi div theta (conservative upwind form).
    """
    d = len(spacing)
    out = np.zeros_like(f)
    for k in range(d):
        axis = d - 1 - k
        n = f.shape[axis]
        lo = [slice(None)] * f.ndim
        hi = list(lo)
        lo[axis] = slice(0, n - 1)
        hi[axis] = slice(1, n)
        lo, hi = tuple(lo), tuple(hi)
        v = th[..., k]
        vf = 0.5 * (v[lo] + v[hi])
        df = (f[hi] - f[lo]) / spacing[k]
        term = np.zeros_like(f)
        term[lo] -= np.minimum(vf, 0.0) * df
        term[hi] -= np.maximum(vf, 0.0) * df
        first = [slice(None)] * f.ndim
        last = list(first)
        first[axis] = 0
        last[axis] = n - 1
        term[tuple(first)] *= 2.0
        term[tuple(last)] *= 2.0
        out += term
    return out


def transport(grid, phi, theta, t_end, steps, smooth, h):
    """Return (new phi, nsub): forward Euler on face-upwind advection
    (+ h^2 lap phi when ``smooth``) with ``nsub`` CFL substeps."""
    if t_end <= 0.0 or steps < 1:
        raise ValueError("transport needs t_end > 0 and steps >= 1")
    d = grid.dim
    shape = _shape(grid)
    nsub, _ = transport_substeps(grid, theta, t_end, steps, smooth, h)
    dt = t_end / nsub
    f = np.asarray(phi, dtype=float).reshape(shape).copy()
    th = np.asarray(theta, dtype=float).reshape(shape + (d,))
    spacing = grid.spacing
    for _ in range(nsub):
        upd = _face_upwind(f, th, spacing)
        if smooth:
            upd = upd + h * h * _laplacian(f, spacing)
        f = f + dt * upd
    return f.reshape(-1), nsub


def reinit_substeps(grid, iters, t_final, h):
    spacing = grid.spacing
    speed = sum(1.0 / s for s in spacing)
    kappa = h * h * sum(2.0 / (s * s) for s in spacing)
    return max(int(iters), int(math.ceil(t_final * (speed + kappa) / CFL)))


def reinitialize(grid, phi, iters, t_final, h):
    """Return (new phi, nsub)."""
    if iters < 2 or t_final <= 0.0:
        raise ValueError("reinitialization needs iters >= 2 and t_final > 0")
    d = grid.dim
    shape = _shape(grid)
    nsub = reinit_substeps(grid, iters, t_final, h)
    dt = t_final / nsub
    f = np.asarray(phi, dtype=float).reshape(shape).copy()
    s = f / np.sqrt(f * f + h * h)
    pos = s > 0.0
    spacing = grid.spacing
    for _ in range(nsub):
        g2 = np.zeros_like(f)
        for k in range(d):
            axis = d - 1 - k
            a, b = _diffs(f, axis, spacing[k])
            gp = np.maximum(np.maximum(a, 0.0) ** 2, np.minimum(b, 0.0) ** 2)
            gn = np.maximum(np.minimum(a, 0.0) ** 2, np.maximum(b, 0.0) ** 2)
            g2 += np.where(pos, gp, gn)
        upd = -s * (np.sqrt(g2) - 1.0) + h * h * _laplacian(f, spacing)
        f = f + dt * upd
    return f.reshape(-1), nsub


# -- the reference's own scheme (restating reference ``levelset.py:109-216``) ----


def _p1_tables(grid):
    """Per-triangle gradients (E,3,2), areas (E,) and the edge-midpoint rule."""
    from .fem import Space, QUAD_BARY_2D
    s = Space(grid, 1)
    return s, s.grads, s.measures, QUAD_BARY_2D


def transport_tau(speed_sq, dt, h):
    """tau = (1/2) (1/dt^2 + |v|^2/h^2)^(-1/2) (``levelset.py:121-127``)."""
    return 0.5 / np.sqrt(1.0 / dt ** 2 + np.asarray(speed_sq) / h ** 2)


def gradient_norm_guard(p):
    """p / sqrt(|p|^2 + eps^2), eps = 1e-12 (1 + |p|) (``levelset.py:109-118``)."""
    p = np.asarray(p, dtype=float)
    mag = np.sqrt(np.sum(p * p, axis=-1, keepdims=True))
    eps = 1e-12 * (1.0 + mag)
    return p / np.sqrt(mag * mag + eps * eps)


def transport_pg(grid, phi, theta, t_end, steps, smooth, h):
    """Crank-Nicolson Petrov-Galerkin transport (``levelset.py:137-169``), 2D."""
    import scipy.sparse.linalg as spla
    space, g, areas, bary = _p1_tables(grid)
    dt = t_end / steps
    th = np.asarray(theta, dtype=float).reshape(-1, 2)[grid.elements]  # (E,3,2)
    th_q = np.einsum("qi,tic->tqc", bary, th)
    tau = transport_tau(np.sum(th_q * th_q, axis=2), dt, h)
    conv = np.einsum("tqd,tid->tqi", th_q, g)
    hat = bary[None, :, :] + tau[:, :, None] * conv
    w = space.quad_weights
    m_hat = np.einsum("tq,tqa,qb->tab", w, hat, bary)
    half = 0.5 * np.einsum("tq,tqa,tqb->tab", w, hat, conv)
    if smooth:
        half = half + 0.5 * h * h * np.einsum("t,tad,tbd->tab", areas, g, g)
    lhs = space.assemble_matrix(m_hat + dt * half)
    rhs = space.assemble_matrix(m_hat - dt * half)
    lu = spla.splu(lhs.tocsc())
    vals = np.asarray(phi, dtype=float).copy()
    for _ in range(steps):
        vals = lu.solve(rhs @ vals)
    return vals


def reinitialize_pg(grid, phi, iters, t_final, h):
    """Petrov-Galerkin Euler/AB2 reinitialisation (``levelset.py:172-216``), 2D."""
    import scipy.sparse.linalg as spla
    space, g, areas, bary = _p1_tables(grid)
    dt = t_final / iters
    phi = np.asarray(phi, dtype=float)
    s_q = np.einsum("qi,ti->tq", bary, phi[grid.elements])
    s_q = s_q / np.sqrt(s_q * s_q + h * h)
    tau = transport_tau(s_q * s_q, dt, h)
    w = space.quad_weights
    cur = phi.copy()
    grad_cur = space.grad_at_quad(cur)
    grad_prev = grad_cur
    for _ in range(iters):
        direction = gradient_norm_guard(grad_cur)
        vel = s_q[:, :, None] * direction[:, None, :]
        conv = np.einsum("tqd,tid->tqi", vel, g)
        hat = bary[None, :, :] + tau[:, :, None] * conv
        m_hat = space.assemble_matrix(np.einsum("tq,tqa,qb->tab", w, hat, bary))
        lu = spla.splu(m_hat.tocsc())
        mag_cur = np.linalg.norm(grad_cur, axis=1)
        mag_prev = np.linalg.norm(grad_prev, axis=1)
        hamiltonian = 0.5 * s_q * (mag_prev - 3.0 * mag_cur)[:, None]
        load = np.einsum("tq,tqa->ta", w * (hamiltonian + s_q), hat)
        diffusion = 0.5 * h * h * np.einsum("t,td,tad->ta", areas, grad_prev - 3.0 * grad_cur, g)
        rhs = m_hat @ cur + dt * space.assemble_vector(load + diffusion)
        cur = lu.solve(rhs)
        grad_prev = grad_cur
        grad_cur = space.grad_at_quad(cur)
    return cur


# -- diagnostics (restating reference ``levelset.py:222-278``) -----------------


def zero_contour_segments(grid, phi):
    """Marching-triangles zero set of a 2D P1 field, (n, 2, 2) segments."""
    tri = grid.elements
    vals = np.asarray(phi)[tri]
    pts = grid.vertices[tri]
    nt = len(vals)
    cand = np.zeros((nt, 6, 2))
    valid = np.zeros((nt, 6), dtype=bool)
    for k, (i, j) in enumerate(((0, 1), (1, 2), (2, 0))):
        a, b = vals[:, i], vals[:, j]
        cross = a * b < 0.0
        t = np.zeros(nt)
        t[cross] = a[cross] / (a[cross] - b[cross])
        cand[:, k] = pts[:, i] + t[:, None] * (pts[:, j] - pts[:, i])
        valid[:, k] = cross
    for v in range(3):
        cand[:, 3 + v] = pts[:, v]
        valid[:, 3 + v] = vals[:, v] == 0.0
    keep = valid.sum(axis=1) == 2
    order = np.argsort(~valid[keep], axis=1, kind="stable")[:, :2]
    return np.take_along_axis(cand[keep], order[:, :, None], axis=1)


def _directed_gap(a, b):
    probes = np.concatenate([a[:, 0], a[:, 1], 0.5 * (a[:, 0] + a[:, 1])])
    start, span = b[:, 0], b[:, 1] - b[:, 0]
    span_sq = np.sum(span * span, axis=1)
    offset = probes[:, None, :] - start[None, :, :]
    t = np.einsum("mnd,nd->mn", offset, span)
    t = np.divide(t, span_sq[None, :], out=np.zeros_like(t), where=span_sq > 0.0)
    np.clip(t, 0.0, 1.0, out=t)
    nearest = start[None, :, :] + t[:, :, None] * span[None, :, :]
    return float(np.linalg.norm(probes[:, None, :] - nearest, axis=2).min(axis=1).max())


def zero_set_displacement(a, b):
    if len(a) == 0 or len(b) == 0:
        return math.inf
    return max(_directed_gap(a, b), _directed_gap(b, a))

"""Compliance model, velocity solve and PPL multipliers (oracle; test infrastructure only).

Restates, dimension-generically:

* ``MaterialIndicator.at_quad`` (reference ``models/base.py:100-121``):
  A_q = chi_q + ersatz (1 - chi_q), chi_q = [phi(x_q) < 0];
* ``ComplianceModel`` / ``CompliancePlusModel`` (``models/compliance.py:37-156``):
  one shared elasticity operator for all loads (``:97-106``), adjoint -2u
  (``:108-109``), J = sum_k int A sigma_k : eps_k (``:111-123``),
  C = int chi / V (``base.py:150-152``), S1 = A sum_k (2 G_k^T sigma_k -
  (sigma_k : eps_k) I) (``:128-139``) plus the multiplier-weighted volume
  tensor lam chi/V I (``base.py:155-158``, ``ppl.py:66-97``);
* ``VelocitySolver`` (``velocity.py:91-154``): B = mass_w M + stiff_w K
  (+ boundary-normal penalty, + frozen mass, + zero Dirichlet), RHS
  vec_a = int S0 . N_a + S1 : grad(N_a e_c), theta = B^-1 (-vec),
  form_value = theta^T B theta, derivative = vec . theta;
* PPL recursion and Lagrangian (``ppl.py:47-63,100-114``);
* ``HeatModel`` / ``HeatPlusModel`` (``models/heat.py:78-171``): two-phase
  conductivity A_q (contrast 1e-3, ``:34,113-114``), one grounded solve per
  term (``:59-76,116-122``), adjoint -c_t u_t (``:124-128``),
  J = sum_t c_t int A |grad u_t|^2 (``:130-138``), S0 = sum_t c_t 2 u grad f,
  S1 = sum_t c_t ((2 u f - A |grad u|^2) I + 2 A grad u (x) grad u)
  (``:143-166``);
* ``InverseElasticityModel`` (``models/inverse.py:78-279``): A_q = kappa chi
  + (1 - chi) (``:102``), forced states (partial clamp) and lifted
  corrections v in H^1_0 with rhs -K g (``:160-178``), misfit, adjoint
  right-hand sides and J (``:180-233``), strain projections (``:142-155``),
  S0/S1 (``:235-279``); ``dirichlet_extension`` and
  ``generate_measurements`` (``:282-353``).
"""

from dataclasses import dataclass, replace

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import fem


class Compliance:
    def __init__(self, grid, lame, ersatz, clamp_dofs, loads, volume):
        self.grid = grid
        self.space = fem.Space(grid, grid.dim)
        self.scalar = fem.Space(grid, 1)
        self.lame = tuple(float(v) for v in lame)
        self.ersatz = float(ersatz)
        self.clamp = np.asarray(clamp_dofs, dtype=np.int64)
        self.loads = [np.asarray(b, dtype=float) for b in loads]
        self.volume = float(volume)

    # -- material -----------------------------------------------------------------
    def chi(self, phi):
        return fem.phi_at_quad_sign(self.space, phi).astype(float)

    def a_q(self, phi):
        chi = self.chi(phi)
        return chi + self.ersatz * (1.0 - chi)

    # -- state ----------------------------------------------------------------------
    def matrix(self, phi):
        a_q = self.a_q(phi)
        return self.space.assemble_matrix_by_parts(
            lambda part: fem.elasticity_elements(part, a_q[part.sl], self.lame))

    def eliminated(self, phi):
        K = self.matrix(phi)
        out = []
        for b in self.loads:
            A, rhs = fem.dirichlet_eliminate(K, b, self.clamp)
            out.append((A, rhs))
        return out

    def solve_states(self, phi, warm=None, rtol=fem.CG_RTOL):
        states, iters = [], []
        for k, (A, b) in enumerate(self.eliminated(phi)):
            x0 = None if warm is None else warm[k]
            x, it = fem.jacobi_pcg(A, b, x0=x0, rtol=rtol)
            states.append(x)
            iters.append(it)
        return states, iters

    # -- functionals ----------------------------------------------------------------
    def energy(self, u):
        jac = self.space.grad_at_quad(u)
        eps = fem.strain(jac)
        sig = fem.stress(eps, self.lame)
        return jac, sig, np.einsum("tij,tij->t", sig, eps)

    def cost(self, phi, states):
        a_q = self.a_q(phi)
        total = 0.0
        for u in states:
            dens = self.energy(u)[2]
            total += float(np.sum(self.space.quad_weights * (a_q * dens[:, None])))
        return total

    def constraint(self, phi):
        return float(np.sum(self.space.quad_weights * self.chi(phi))) / self.volume

    def s1_cost(self, phi, states):
        a_q = self.a_q(phi)
        d = self.grid.dim
        s1 = np.zeros(a_q.shape + (d, d))
        for u in states:
            jac, sig, dens = self.energy(u)
            bulk = 2.0 * np.einsum("tki,tkj->tij", jac, sig) - dens[:, None, None] * np.eye(d)
            s1 += a_q[:, :, None, None] * bulk[:, None, :, :]
        return s1

    def s1_volume(self, phi):
        return self.chi(phi)[:, :, None, None] * (np.eye(self.grid.dim) / self.volume)

    def s1_combined(self, phi, states, lam):
        return self.s1_cost(phi, states) + lam * self.s1_volume(phi)


class Heat:
    """Summed thermal compliance with a volume constraint (reference ``models/heat.py``).

    ``terms`` = [(weight, ground node list, f_q (E, 3), gradf_q (E, 3, 2) or None)];
    a None weight means 1 / len(terms) (``heat.py:107-111``).
    """

    CONTRAST = 1e-3

    def __init__(self, grid, terms, volume, contrast=CONTRAST):
        self.grid = grid
        self.space = fem.Space(grid, 1)
        self.contrast = float(contrast)
        self.volume = float(volume)
        default_w = 1.0 / len(terms)
        self.terms = []
        for w, ground, f_q, g_q in terms:
            load = self.space.assemble_vector(
                np.einsum("tq,qa->ta", self.space.quad_weights * f_q, self.space.bary))
            self.terms.append((default_w if w is None else float(w), np.asarray(ground, dtype=np.int64),
                               np.asarray(f_q, dtype=float), None if g_q is None else np.asarray(g_q, dtype=float),
                               load))

    def chi(self, phi):
        return fem.phi_at_quad_sign(self.space, phi).astype(float)

    def a_q(self, phi):
        chi = self.chi(phi)
        return chi + self.contrast * (1.0 - chi)

    def matrix(self, phi):
        return self.space.assemble_matrix(fem.stiffness_elements(self.space, self.a_q(phi)))

    def solve_states(self, phi, rtol=fem.CG_RTOL):
        K = self.matrix(phi)
        states, iters = [], []
        for _, ground, _, _, load in self.terms:
            A, b = fem.dirichlet_eliminate(K, load, ground)
            x, it = fem.jacobi_pcg(A, b, rtol=rtol)
            states.append(x)
            iters.append(it)
        return states, iters

    def cost(self, phi, states):
        a_q = self.a_q(phi)
        total = 0.0
        for (w, *_), u in zip(self.terms, states):
            g = self.space.grad_at_quad(u)
            dens = np.einsum("td,td->t", g, g)
            total += w * float(np.sum(self.space.quad_weights * (a_q * dens[:, None])))
        return total

    def constraint(self, phi):
        return float(np.sum(self.space.quad_weights * self.chi(phi))) / self.volume

    def tensors(self, phi, states):
        """(S0, S1) of the cost at the quadrature points (``heat.py:143-166``)."""
        a_q = self.a_q(phi)
        nt, nq = a_q.shape
        s0 = np.zeros((nt, nq, 2))
        s1 = np.zeros((nt, nq, 2, 2))
        for (w, _, f_q, g_q, _), u in zip(self.terms, states):
            u_q = np.einsum("qa,ta->tq", self.space.bary, u[self.grid.elements])
            g = self.space.grad_at_quad(u)
            dens = np.einsum("td,td->t", g, g)
            if g_q is not None:
                s0 += w * 2.0 * u_q[:, :, None] * g_q
            scal = 2.0 * u_q * f_q - a_q * dens[:, None]
            outer = np.einsum("ti,tj->tij", g, g)
            s1 += w * (scal[:, :, None, None] * np.eye(2) + 2.0 * a_q[:, :, None, None] * outer[:, None, :, :])
        return s0, s1


EDGE_GAUSS = np.array([0.5 - 0.5 / np.sqrt(3.0), 0.5 + 0.5 / np.sqrt(3.0)])
EDGE_BASIS = np.stack([1.0 - EDGE_GAUSS, EDGE_GAUSS], axis=1)


def _facet_mass_vector(grid, facet_ids, values):
    """sum_f int_f (vector field) N_a with the 2-point Gauss rule (``fem.py:441-448``)."""
    facets = grid.boundary_facets[facet_ids]
    lengths = grid.facet_measures()[facet_ids]
    nodal = np.asarray(values).reshape(-1, 2)[facets]  # (nf, 2 nodes, 2 comps)
    tr = np.einsum("qi,fic->fqc", EDGE_BASIS, nodal)
    elems = np.einsum("fq,fqc,qa->fac", np.repeat((lengths / 2.0)[:, None], 2, axis=1), tr, EDGE_BASIS)
    out = np.zeros(2 * grid.num_vertices)
    dofs = 2 * facets[:, :, None] + np.arange(2)[None, None, :]
    np.add.at(out, dofs.reshape(len(facets), -1), elems.reshape(len(facets), -1))
    return out, tr, lengths


class Inverse:
    """Kohn-Vogelius inclusion recovery (reference ``models/inverse.py``), 2D."""

    def __init__(self, grid, partial_dofs, measured_facets, loads, measured, contrast=10.0,
                 alpha=1.0, beta=1.0, lame=(1.25, 1.0)):
        self.grid = grid
        self.space = fem.Space(grid, 2)
        self.scalar = fem.Space(grid, 1)
        self.partial = np.asarray(partial_dofs, dtype=np.int64)
        self.total = fem.clamp_dofs(self.space, np.arange(len(grid.boundary_facets)))
        self.mfacets = np.asarray(measured_facets, dtype=np.int64)
        self.loads = [np.asarray(b, dtype=float) for b in loads]
        self.g = [np.asarray(v, dtype=float) for v in measured]
        self.contrast, self.alpha, self.beta = float(contrast), float(alpha), float(beta)
        self.lame = tuple(float(v) for v in lame)
        mass = self.scalar.assemble_matrix(fem.mass_elements(self.scalar))
        self.proj = [self._project(mass, g) for g in self.g]

    def _project(self, mass, g):
        """Gradients of the nodal projections of eps(g): (E, 2, 2, 2) (``inverse.py:142-155``)."""
        eps = fem.strain(self.space.grad_at_quad(g))
        nt, nq = self.scalar.quad_weights.shape
        out = np.empty((nt, 2, 2, 2))
        for i, j in ((0, 0), (0, 1), (1, 1)):
            comp_q = np.broadcast_to(eps[:, i, j][:, None], (nt, nq))
            rhs = self.scalar.assemble_vector(np.einsum("tq,qa->ta", self.scalar.quad_weights * comp_q,
                                                        self.scalar.bary))
            nodal, _ = fem.jacobi_pcg(mass, rhs)
            out[:, i, j, :] = self.scalar.grad_at_quad(nodal)
        out[:, 1, 0, :] = out[:, 0, 1, :]
        return out

    def a_q(self, phi):
        chi = fem.phi_at_quad_sign(self.space, phi).astype(float)
        return self.contrast * chi + (1.0 - chi)

    def matrix(self, phi):
        return self.space.assemble_matrix(fem.elasticity_elements(self.space, self.a_q(phi), self.lame))

    def state_systems(self, phi):
        K = self.matrix(phi)
        forced = [fem.dirichlet_eliminate(K, b, self.partial) for b in self.loads]
        lifted = [fem.dirichlet_eliminate(K, -(K @ g), self.total) for g in self.g]
        return forced + lifted

    def solve(self, systems):
        return [fem.jacobi_pcg(A, b)[0] for A, b in systems]

    def misfit(self, states):
        n = len(self.g)
        out = []
        for g, u, v in zip(self.g, states[:n], states[n:]):
            e = u - v - g
            me = self.space.assemble_vector(np.einsum(
                "tq,tqc,qa->tac", self.space.quad_weights,
                np.einsum("qi,tic->tqc", self.space.bary, e.reshape(-1, 2)[self.grid.elements]),
                self.space.bary).reshape(len(self.grid.elements), -1))
            mf, tr, lengths = _facet_mass_vector(self.grid, self.mfacets, u - g)
            out.append((e, me, u - g, mf))
        return out

    def cost(self, states):
        total = 0.0
        for e, me, f, mf in self.misfit(states):
            total += 0.5 * self.alpha * float(e @ me) + 0.5 * self.beta * float(f @ mf)
        return total

    def adjoint_systems(self, phi, states):
        K = self.matrix(phi)
        mis = self.misfit(states)
        head = [fem.dirichlet_eliminate(K, -self.alpha * me - self.beta * mf, self.partial)
                for _, me, _, mf in mis]
        tail = [fem.dirichlet_eliminate(K, self.alpha * me, self.total) for _, me, _, _ in mis]
        return head + tail

    def tensors(self, phi, states, adjoints):
        a_q = self.a_q(phi)
        n = len(self.g)
        nt, nq = a_q.shape
        s0 = np.zeros((nt, nq, 2))
        s1 = np.zeros((nt, nq, 2, 2))
        sp_ = self.space
        for k in range(n):
            u, v, g = states[k], states[n + k], self.g[k]
            p, q = adjoints[k], adjoints[n + k]
            bulk = np.einsum("qi,tic->tqc", sp_.bary, (u - v - g).reshape(-1, 2)[self.grid.elements])
            ju, jv, jp, jq, jg = (sp_.grad_at_quad(x) for x in (u, v, p, q, g))
            su, spp, sq = (fem.stress(fem.strain(j), self.lame) for j in (ju, jp, jq))
            sy = fem.stress(fem.strain(jv + jg), self.lame)
            s0 -= self.alpha * np.einsum("tji,tqj->tqi", jg, bulk)
            drift = np.einsum("tij,tijk->tk", sq, self.proj[k])
            s0 += a_q[:, :, None] * drift[:, None, :]
            scal = 0.5 * self.alpha * np.einsum("tqc,tqc->tq", bulk, bulk)
            pairing = (np.einsum("tij,tij->t", su, fem.strain(jp))
                       + np.einsum("tij,tij->t", sy, fem.strain(jq)))
            scal = scal + a_q * pairing[:, None]
            mat = (np.einsum("tki,tkj->tij", ju, spp) + np.einsum("tki,tkj->tij", jp, su)
                   + np.einsum("tki,tkj->tij", jv, sq) + np.einsum("tki,tkj->tij", jq, sy))
            s1 += scal[:, :, None, None] * np.eye(2)
            s1 -= a_q[:, :, None, None] * mat[:, None, :, :]
        return s0, s1


def dirichlet_extension(grid, facet_ids, traces):
    """Harmonic extension (``inverse.py:282-313``): vector Laplace, values on the facet nodes."""
    space = fem.Space(grid, 2)
    nodes = np.unique(grid.boundary_facets[facet_ids])
    dofs = np.column_stack([2 * nodes, 2 * nodes + 1]).reshape(-1)
    K = space.assemble_matrix(fem.stiffness_elements(space))
    out = []
    for tr in traces:
        A, b = fem.dirichlet_eliminate(K, np.zeros(space.dof_count), dofs, np.asarray(tr)[dofs])
        out.append(fem.jacobi_pcg(A, b)[0])
    return out


def derivative_vector(space, s1=None, s0=None):
    """vec_(a,c) = int S0_c N_a + S1[c,:] . grad N_a (reference ``velocity.py:129-142``)."""
    vec = np.zeros(space.dof_count)
    n_el = len(space.grads)
    if s0 is not None:
        elems = np.einsum("tq,tqc,qa->tac", space.quad_weights, s0, space.bary)
        vec += space.assemble_vector(elems.reshape(n_el, -1))
    if s1 is not None:
        elems = np.einsum("tq,tqcd,tad->tac", space.quad_weights, s1, space.grads)
        vec += space.assemble_vector(elems.reshape(n_el, -1))
    return vec


def facet_normal_axes(grid):
    """Outward normal of each boundary facet of the box as (axis, sign)."""
    mids = grid.facet_midpoints()
    axes = np.zeros(len(mids), dtype=np.int64)
    signs = np.zeros(len(mids))
    for a in range(grid.dim):
        lo = np.isclose(mids[:, a], grid.lo[a], rtol=0, atol=1e-12 * (grid.hi[a] - grid.lo[a]))
        hi = np.isclose(mids[:, a], grid.hi[a], rtol=0, atol=1e-12 * (grid.hi[a] - grid.lo[a]))
        axes[lo | hi] = a
        signs[lo] = -1.0
        signs[hi] = 1.0
    return axes, signs


class Velocity:
    """H1-type velocity form, solved by sparse LU (reference ``velocity.py:98-127``)."""

    def __init__(self, grid, mass_weight=1.0, stiffness_weight=1e-2,
                 boundary_normal_penalty=0.0, frozen_chi=None, frozen_penalty=0.0,
                 zero_dirichlet=False, direct=True):
        # direct=False: Jacobi-CG to a 1e-14 relative residual instead of SuperLU
        # (test-fixture generation on large 3D grids, where the LU fill of a 3D
        # form is out of reach; the form is SPD and well conditioned, the two
        # agree to ~1e-13, far inside every gate that uses theta)
        self.direct = direct
        self.grid = grid
        self.space = fem.Space(grid, grid.dim)
        sp_ = self.space
        def form_elements(part):
            elems = stiffness_weight * fem.stiffness_elements(part)
            if mass_weight > 0:
                elems = elems + mass_weight * fem.mass_elements(part)
            if frozen_chi is not None and frozen_penalty > 0:
                elems = elems + frozen_penalty * fem.mass_elements(part, np.asarray(frozen_chi)[part.sl])
            return elems

        B = sp_.assemble_matrix_by_parts(form_elements)
        if boundary_normal_penalty > 0:
            B = B + boundary_normal_penalty * self._normal_matrix()
        self.form_matrix = B.tocsr()
        self.bc = None
        solvable = self.form_matrix
        if zero_dirichlet:
            self.bc = fem.clamp_dofs(sp_, np.arange(len(grid.boundary_facets)))
            solvable, _ = fem.dirichlet_eliminate(self.form_matrix, np.zeros(sp_.dof_count), self.bc)
        self.solvable = solvable.tocsr()
        self.lu = spla.splu(solvable.tocsc()) if direct else None

    def _normal_matrix(self):
        grid, d = self.grid, self.grid.dim
        facets = grid.boundary_facets
        meas = grid.facet_measures()
        axes, _ = facet_normal_axes(grid)
        nv = d  # vertices per facet
        local = (np.ones((nv, nv)) + np.eye(nv)) / (nv * (nv + 1))
        rows, cols, vals = [], [], []
        for a in range(nv):
            for b in range(nv):
                rows.append(d * facets[:, a] + axes)
                cols.append(d * facets[:, b] + axes)
                vals.append(meas * local[a, b])
        n = self.space.dof_count
        return sp.coo_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                             shape=(n, n)).tocsr()

    def solve(self, vec):
        rhs = -vec
        if self.bc is not None:
            rhs = rhs.copy()
            rhs[self.bc] = 0.0
        theta = self.lu.solve(rhs) if self.direct else _jacobi_cg(self.solvable, rhs, 1e-14)
        return theta, float(theta @ (self.form_matrix @ theta)), float(vec @ theta)


def _jacobi_cg(A, b, rtol, maxiter=20000):
    """Plain Jacobi-preconditioned CG (numpy), stopping at ||r|| <= rtol ||b||."""
    dinv = 1.0 / A.diagonal()
    x = np.zeros_like(b)
    r = b.copy()
    z = dinv * r
    p = z.copy()
    rz = float(r @ z)
    stop = rtol * float(np.linalg.norm(b))
    for _ in range(maxiter):
        if float(np.linalg.norm(r)) <= stop:
            break
        q = A @ p
        alpha = rz / float(p @ q)
        x += alpha * p
        r -= alpha * q
        z = dinv * r
        rz, rz_old = float(r @ z), rz
        p = z + (rz / rz_old) * p
    return x


@dataclass(frozen=True)
class Ppl:
    z: np.ndarray
    lam: np.ndarray
    mu: np.ndarray
    delta: float = 0.5
    r: float = 0.999
    alpha: float = 2000.0
    beta: float = 0.5


def ppl_init(nc):
    return Ppl(np.zeros(nc), np.zeros(nc), np.zeros(nc))


def ppl_update(s, c):
    c = np.asarray(c, dtype=float).reshape(-1)
    gap = s.lam - s.mu
    mu = s.mu + s.delta * gap / (float(gap @ gap) + 1.0)
    lam = mu + s.alpha / (1.0 + s.alpha * s.beta) * (c - 1.0)
    z = (lam - mu) / s.alpha
    return replace(s, z=z, lam=lam, mu=mu, delta=s.r * s.delta)


def lagrangian(cost, c, s):
    c = np.asarray(c, dtype=float).reshape(-1)
    gap = s.lam - s.mu
    return float(cost + s.lam @ (c - 1.0) + s.mu @ s.z
                 + 0.5 * s.alpha * float(s.z @ s.z) + 0.5 * s.beta * float(gap @ gap))

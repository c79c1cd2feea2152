"""The CPU oracle against the reference's golden vectors (pins the oracle).

Golden vectors come from the reference itself (tests/golden/make_golden.py);
the explicit level-set scheme, which has no reference implementation, is
pinned by the reference's scheme-agnostic property tests
(reference tests/test_levelset.py:155-286) re-run on the oracle.
"""

import math

import numpy as np
import pytest

from conftest import rel_l2
from oracle import fem, levelset
from oracle.grid import Grid, level_set_h, mesh_diameter
from oracle.model import Compliance, Velocity, derivative_vector, lagrangian, ppl_init, ppl_update
from oracle import driver as odriver

LAME = (0.3 / 0.91, 1.0 / 2.6)


def cantilever_grid(nx, ny):
    rules = [(1, lambda p: p[:, 0] < 1e-12),
             (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55))]
    return Grid((0.0, 0.0), (2.0, 1.0), (nx, ny), rules)


def phi_fn(p):
    return -np.cos(6 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) - 0.4


@pytest.fixture(scope="module")
def setup32():
    grid = cantilever_grid(32, 16)
    space = fem.Space(grid, 2)
    clamp = fem.clamp_dofs(space, grid.facets_with_tag(1))
    load = fem.boundary_traction_vector(space, grid.facets_with_tag(2), (0.0, -1.0))
    model = Compliance(grid, LAME, 1e-3, clamp, [load], 1.0)
    phi = phi_fn(grid.vertices)
    return grid, space, model, phi


class TestMeshKAT:
    def test_connectivity_bit_exact(self, golden):
        g = cantilever_grid(7, 5)
        np.testing.assert_array_equal(g.vertices, golden["mesh_vertices"])
        np.testing.assert_array_equal(g.elements, golden["mesh_triangles"])
        np.testing.assert_array_equal(g.boundary_facets, golden["mesh_facets"])
        np.testing.assert_array_equal(g.facet_tags, golden["mesh_tags"])
        assert mesh_diameter(g) == golden["mesh_diameter_7x5"][0]

    def test_odd_bounds_linspace(self, golden):
        g = Grid((-0.3, 0.1), (1.7, 1.3), (13, 9))
        np.testing.assert_array_equal(g.vertices, golden["odd_vertices"])


class TestOperatorKAT:
    def test_indicator_bit_exact(self, golden, setup32):
        grid, space, model, phi = setup32
        np.testing.assert_array_equal(phi, golden["phi_32x16"])
        np.testing.assert_array_equal(model.chi(phi), golden["chi_32x16"])
        assert level_set_h(grid) == pytest.approx(golden["h_32x16"][0], rel=1e-15)

    def test_apply_and_elimination(self, golden, setup32):
        grid, space, model, phi = setup32
        K = model.matrix(phi)
        for u, ku in zip(golden["apply_u"], golden["apply_Ku"]):
            assert rel_l2(K @ u, ku) <= 1e-13
        Ke, _ = fem.dirichlet_eliminate(K, np.zeros(space.dof_count), model.clamp)
        for u, ku in zip(golden["apply_u"], golden["apply_Keu"]):
            assert rel_l2(Ke @ u, ku) <= 1e-13
        np.testing.assert_array_equal(model.clamp, golden["bc_dofs"])
        assert rel_l2(Ke.diagonal(), golden["diag_elim"]) <= 1e-14

    def test_loads(self, golden, setup32):
        grid, space, model, phi = setup32
        assert rel_l2(model.loads[0], golden["load_vector"]) <= 1e-15
        bf = fem.body_force_vector(space, (0.0, -1.0))
        assert rel_l2(bf, golden["body_force_vector"]) <= 1e-14


class TestComplianceKAT:
    def test_state_cost_constraint(self, golden, setup32):
        grid, space, model, phi = setup32
        states, iters = model.solve_states(phi)
        assert rel_l2(states[0], golden["state_u"]) <= 1e-8
        assert model.cost(phi, states) == pytest.approx(golden["J"][0], rel=1e-10)
        assert model.constraint(phi) == pytest.approx(golden["C"][0], rel=1e-14)
        assert iters[0] > 10

    def test_s1_and_velocity(self, golden, setup32):
        grid, space, model, phi = setup32
        states = [golden["state_u"]]
        assert rel_l2(model.s1_cost(phi, states), golden["S1_cost"]) <= 1e-12
        lam = 0.37
        vec = derivative_vector(space, s1=model.s1_combined(phi, states, lam))
        assert rel_l2(vec, golden["velocity_vec"]) <= 1e-12
        vel = Velocity(grid, 1.0, 1e-2)
        theta, btt, dj = vel.solve(vec)
        assert rel_l2(theta, golden["theta"]) <= 1e-10
        assert btt == pytest.approx(golden["form_value"][0], rel=1e-10)
        assert dj == pytest.approx(golden["derivative"][0], rel=1e-10)

    @pytest.mark.parametrize("name,kw", [
        ("normal", dict(mass_weight=0.1, stiffness_weight=1.0, boundary_normal_penalty=1e4)),
        ("dirichlet", dict(mass_weight=0.0, stiffness_weight=1.0, zero_dirichlet=True)),
        ("frozen", dict(mass_weight=1.0, stiffness_weight=0.5, frozen_penalty=1e2)),
    ])
    def test_velocity_form_variants(self, golden, setup32, name, kw):
        grid, space, model, phi = setup32
        if name == "frozen":
            kw["frozen_chi"] = (space.quad_points[..., 0] > 1.6).astype(float)
        vel = Velocity(grid, **kw)
        assert rel_l2(vel.form_matrix @ golden["apply_u"][0], golden[f"form_apply_{name}"]) <= 1e-13
        theta, btt, _ = vel.solve(golden["velocity_vec"])
        assert rel_l2(theta, golden[f"theta_{name}"]) <= 1e-9
        assert btt == pytest.approx(golden[f"form_value_{name}"][0], rel=1e-9)

    def test_two_loads(self, golden, setup32):
        grid, space, model, phi = setup32
        l2 = fem.boundary_traction_vector(space, grid.facets_with_tag(2), (0.0, -2.0))
        plus = Compliance(grid, LAME, 1e-3, model.clamp, [model.loads[0], l2], 1.0)
        states, _ = plus.solve_states(phi)
        assert rel_l2(np.stack(states), golden["plus_states"]) <= 1e-8
        assert plus.cost(phi, states) == pytest.approx(golden["plus_J"][0], rel=1e-9)


class TestReferenceScheme:
    """The reference's CN/PG transport and PG/AB2 reinit (levelset.py:137-216), restated."""

    def test_transport_and_reinit(self, golden):
        g = Grid((0.0, 0.0), (1.0, 1.0), (24, 20))
        h = level_set_h(g)
        for smooth, key in ((False, "ls_transport"), (True, "ls_transport_smooth")):
            out = levelset.transport_pg(g, golden["ls_phi"], golden["ls_theta"], 0.03, 8, smooth, h)
            assert rel_l2(out, golden[key]) <= 1e-13
        out = levelset.reinitialize_pg(g, 3.0 * golden["ls_phi"], 8, 0.1, h)
        assert rel_l2(out, golden["ls_reinit"]) <= 1e-13

    def test_full_loop_matches_reference_run(self, golden):
        """Oracle loop with the reference scheme vs the reference's own run()
        (cfg1 geometry at 40x20, 12 iterations, reinit every 5)."""
        from oracle import cases as ocases
        from paper_2601_05709_b200 import configs
        c = configs.case("cfg1", scale=4)
        c = type(c)(**{**c.__dict__, "niter": 12, "reinit_step": 5})
        grid, om, ovel, phi0, params, h = ocases.build(c)
        params = odriver.Params(**{**params.__dict__, "scheme": "pg"})
        _, hist = odriver.run(om, ovel, phi0, params, h)
        np.testing.assert_allclose([r["cost"] for r in hist], golden["run_cost"], rtol=1e-8)
        np.testing.assert_allclose([r["constraint"][0] for r in hist], golden["run_constraint"], rtol=1e-12)
        np.testing.assert_allclose([r["lagrangian"] for r in hist], golden["run_lagrangian"], rtol=1e-8)
        np.testing.assert_allclose([r["t_end"] for r in hist], golden["run_t_end"], rtol=1e-8)
        np.testing.assert_array_equal([r["steps"] for r in hist], golden["run_steps"])


class TestHostKAT:
    def test_ppl_table(self, golden):
        st = ppl_init(1)
        for c, row in zip(golden["ppl_inputs"], golden["ppl_table"]):
            st = ppl_update(st, [c])
            got = [st.z[0], st.lam[0], st.mu[0], st.delta, lagrangian(2.0, [c], st)]
            np.testing.assert_allclose(got, row, rtol=1e-15, atol=0)

    def test_adaptive_time_rng_order(self, golden):
        params = odriver.Params()
        rng = np.random.default_rng(1)
        got = [odriver.adaptive_time(b, params, rng) for b in golden["adaptive_btt"]]
        np.testing.assert_array_equal(np.array(got, dtype=float), golden["adaptive_out"])


def unit_square(n):
    return Grid((0.0, 0.0), (1.0, 1.0), (n, n))


def disk(g, c=(0.5, 0.5), r=0.3):
    return np.linalg.norm(g.vertices - np.asarray(c), axis=1) - r


def p1_mass(g, f):
    s = fem.Space(g)
    return float(np.sum(s.quad_weights * np.einsum("qi,ti->tq", s.bary, f[g.elements])))


class TestLevelSetProperties:
    """Reference tests/test_levelset.py:155-286, re-run on the explicit scheme."""

    def test_zero_velocity_identity(self):
        g = unit_square(24)
        phi = disk(g)
        out, _ = levelset.transport(g, phi, np.zeros(2 * g.num_vertices), 5e-2, 5, False, level_set_h(g))
        assert np.max(np.abs(out - phi)) <= 1e-10

    def test_noise_diffusion_dissipates(self):
        g = unit_square(32)
        s = fem.Space(g)
        phi = np.random.default_rng(7).normal(size=g.num_vertices)

        def energy(f):
            gr = s.grad_at_quad(f)
            return float(np.sum(s.measures * np.sum(gr * gr, axis=1)))

        es = [energy(phi)]
        for _ in range(6):
            phi, _ = levelset.transport(g, phi, np.zeros(2 * g.num_vertices), 1.0, 1, True, level_set_h(g))
            es.append(energy(phi))
        assert all(b <= a * (1 + 1e-12) for a, b in zip(es, es[1:]))
        assert es[-1] < 0.999 * es[0]

    def test_disk_radius_growth(self):
        g = unit_square(128)
        phi = disk(g)
        c = np.array([0.5, 0.5])
        d = g.vertices - c
        th = d / np.sqrt(np.sum(d * d, axis=1, keepdims=True) + 0.02 ** 2)
        out, _ = levelset.transport(g, phi, th.ravel(), 0.02, 8, False, level_set_h(g))
        rad = lambda segs: float(np.mean(np.linalg.norm(segs.reshape(-1, 2) - c, axis=1)))
        growth = rad(levelset.zero_contour_segments(g, out)) - rad(levelset.zero_contour_segments(g, phi))
        assert growth == pytest.approx(0.02, rel=0.2)

    def test_mass_drift_divergence_free(self):
        g = unit_square(64)
        phi = disk(g)
        x, y = g.vertices[:, 0], g.vertices[:, 1]
        th = np.stack([math.pi * np.sin(math.pi * x) * np.cos(math.pi * y),
                       -math.pi * np.cos(math.pi * x) * np.sin(math.pi * y)], axis=1)
        out, _ = levelset.transport(g, phi, th.ravel(), 0.5, 100, False, level_set_h(g))
        drift = abs(p1_mass(g, out) - p1_mass(g, phi)) / (abs(p1_mass(g, phi)) * 0.5)
        assert drift < 0.01

    @pytest.mark.parametrize("shape", ["line", "disk"])
    def test_distance_is_fixed_point(self, shape):
        g = unit_square(32)
        h = level_set_h(g)
        phi = g.vertices[:, 0] - 0.5 if shape == "line" else disk(g)
        out, _ = levelset.reinitialize(g, phi, 8, 0.1, h)
        vals = phi[g.elements]
        band = ((vals.min(1) < 0) & (vals.max(1) > 0)) | (np.abs(vals).min(1) <= 3 * h)
        gn = np.linalg.norm(fem.Space(g).grad_at_quad(out), axis=1)
        assert np.max(np.abs(gn[band] - 1.0)) <= 0.1
        moved = levelset.zero_set_displacement(levelset.zero_contour_segments(g, phi),
                                               levelset.zero_contour_segments(g, out))
        assert moved <= 2.0 * h

    def test_rescaled_field_keeps_zero_set(self):
        g = unit_square(32)
        h = level_set_h(g)
        phi = 5.0 * disk(g)
        out, _ = levelset.reinitialize(g, phi, 8, 0.1, h)
        moved = levelset.zero_set_displacement(levelset.zero_contour_segments(g, phi),
                                               levelset.zero_contour_segments(g, out))
        assert moved <= h

    def test_constant_field_grows_linearly(self):
        g = unit_square(20)
        h = level_set_h(g)
        out, _ = levelset.reinitialize(g, np.ones(g.num_vertices), 8, 0.1, h)
        np.testing.assert_allclose(out, 1.0 + 0.1 / math.sqrt(1.0 + h * h), atol=1e-9)


@pytest.fixture(scope="module")
def box():
    g = Grid((0.0, 0.0, 0.0), (2.0, 1.0, 1.0), (4, 3, 2))
    return g, fem.Space(g, 3)


class TestOracle3D:
    """Dimension-generic identities for the 3D restatement (no reference exists)."""


    def test_counts_and_volume(self, box):
        g, s = box
        assert g.num_vertices == 5 * 4 * 3
        assert g.num_elements == 6 * 4 * 3 * 2
        assert s.measures.sum() == pytest.approx(2.0, rel=1e-14)
        assert np.allclose(s.measures, 2.0 / g.num_elements, rtol=1e-12)
        assert g.facet_measures().sum() == pytest.approx(2 * (2 + 2 + 1), rel=1e-14)

    def test_conforming(self, box):
        g, _ = box
        faces = {}
        for t in g.elements:
            for skip in range(4):
                f = tuple(sorted(np.delete(t, skip)))
                faces[f] = faces.get(f, 0) + 1
        boundary = {tuple(sorted(f)) for f in g.boundary_facets}
        for f, cnt in faces.items():
            assert cnt == (1 if f in boundary else 2)

    def test_rigid_motions_in_kernel(self, box):
        g, s = box
        chi = np.random.default_rng(0).random((g.num_elements, 4))
        K = s.assemble_matrix(fem.elasticity_elements(s, chi, (0.57, 0.38)))
        x = g.vertices
        for mode in (np.tile([1, 0, 0], (len(x), 1)), np.stack([-x[:, 1], x[:, 0], 0 * x[:, 0]], 1),
                     np.stack([0 * x[:, 0], -x[:, 2], x[:, 1]], 1)):
            assert np.abs(K @ mode.ravel()).max() <= 1e-12
        assert abs(K - K.T).max() <= 1e-14

    def test_mass_total(self, box):
        g, s = box
        s1 = fem.Space(g, 1)
        M = s1.assemble_matrix(fem.mass_elements(s1))
        assert M.sum() == pytest.approx(2.0, rel=1e-13)


# -- heat models (reference models/heat.py), pinned to tests/golden/reference_heat.npz --------
def _heat_oracle():
    from oracle import model as om
    from oracle.grid import Grid
    from heat_cases import BOUNDS, NX, NY, RULES, grad_a, phi_fn, src_a, src_b
    grid = Grid(BOUNDS[:2], BOUNDS[2:], (NX, NY), RULES)
    space = om.fem.Space(grid, 1)
    pts = space.quad_points.reshape(-1, 2)
    fa = src_a(pts).reshape(-1, 3)
    ga = grad_a(pts).reshape(-1, 3, 2)
    fb = src_b(pts).reshape(-1, 3)
    ground_a = np.unique(grid.boundary_facets[grid.facets_with_tag(1)])
    ground_b = np.unique(grid.boundary_facets[grid.facets_with_tag((2, 3))])
    model = om.Heat(grid, [(0.7, ground_a, fa, ga), (None, ground_b, fb, None)], 0.6)
    return grid, model, phi_fn(grid.vertices)


def test_heat_oracle_matches_reference():
    import os
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_heat.npz"))
    from oracle import model as om
    grid, model, phi = _heat_oracle()
    np.testing.assert_allclose(phi, g["phi"], rtol=0, atol=0)
    np.testing.assert_allclose(np.stack([t[4] for t in model.terms]), g["loads"], rtol=1e-13, atol=1e-16)
    states, _ = model.solve_states(phi)
    for u, ref in zip(states, g["states"]):
        assert np.linalg.norm(u - ref) <= 1e-8 * np.linalg.norm(ref)
    states = list(g["states"])  # evaluate the functionals on the reference states
    assert model.cost(phi, states) == pytest.approx(float(g["J"][0]), rel=1e-12)
    assert model.constraint(phi) == pytest.approx(float(g["C"][0]), rel=1e-14)
    s0, s1 = model.tensors(phi, states)
    np.testing.assert_allclose(s0, g["S0"], rtol=1e-12, atol=1e-13)
    np.testing.assert_allclose(s1, g["S1"], rtol=1e-12, atol=1e-12)
    vspace = om.fem.Space(grid, 2)
    vec = om.derivative_vector(vspace, s1=s1, s0=s0)
    assert np.linalg.norm(vec - g["vec_cost"]) <= 1e-12 * np.linalg.norm(g["vec_cost"])


# -- inverse-elasticity model (reference models/inverse.py), pinned to reference_inverse.npz --
def test_inverse_oracle_matches_reference():
    import os
    from inverse_cases import (BOUNDS, COARSE, CONTRAST, FINE, FIXED, FORCES, LAME, MEASURED,
                               guess, inclusion, rules)
    from oracle import model as om
    g = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_inverse.npz"))
    coarse = Grid(BOUNDS[:2], BOUNDS[2:], COARSE, rules())
    fine = Grid(BOUNDS[:2], BOUNDS[2:], FINE, rules())
    # twin measurements: fine solve with the true inclusion, injection, harmonic extension
    fspace = fem.Space(fine, 2)
    fmodel = om.Inverse(fine, fem.clamp_dofs(fspace, fine.facets_with_tag(FIXED)),
                        fine.facets_with_tag(MEASURED),
                        [fem.boundary_traction_vector(fspace, fine.facets_with_tag(t), tr) for tr, t in FORCES],
                        [np.zeros(fspace.dof_count)], contrast=CONTRAST, lame=LAME)
    K = fmodel.matrix(inclusion(fine.vertices))
    inj = np.array([np.flatnonzero((np.abs(fine.vertices - v) < 1e-12).all(axis=1))[0]
                    for v in coarse.vertices])
    traces = []
    for b in fmodel.loads:
        A, rhs = fem.dirichlet_eliminate(K, b, fmodel.partial)
        traces.append(fem.jacobi_pcg(A, rhs)[0].reshape(-1, 2)[inj].reshape(-1))
    ext = om.dirichlet_extension(coarse, coarse.facets_with_tag((FIXED,) + MEASURED), traces)
    for x, ref in zip(ext, g["measured"]):
        assert rel_l2(x, ref) <= 1e-8
    e2 = om.dirichlet_extension(coarse, coarse.facets_with_tag((1, 3)), [g["ext_trace"]])[0]
    assert rel_l2(e2, g["ext_out"]) <= 1e-9
    # the model pieces on the reference's own inputs
    cspace = fem.Space(coarse, 2)
    model = om.Inverse(coarse, fem.clamp_dofs(cspace, coarse.facets_with_tag(FIXED)),
                       coarse.facets_with_tag(MEASURED),
                       [fem.boundary_traction_vector(cspace, coarse.facets_with_tag(t), tr) for tr, t in FORCES],
                       list(g["measured"]), contrast=CONTRAST, lame=LAME)
    phi = g["phi"]
    np.testing.assert_array_equal(phi, guess(coarse.vertices))
    systems = model.state_systems(phi)
    # the reference's LinearProblem.rhs is the raw right-hand side (before elimination)
    raw = model.loads + [-(model.matrix(phi) @ x) for x in model.g]
    np.testing.assert_allclose(np.stack(raw), g["state_rhs"], rtol=1e-12, atol=1e-14)
    states = model.solve(systems)
    for x, ref in zip(states, g["states"]):
        assert rel_l2(x, ref) <= 1e-8
    states = list(g["states"])
    assert model.cost(states) == pytest.approx(float(g["J"][0]), rel=1e-12)
    mis = model.misfit(states)
    head = [-model.alpha * me - model.beta * mf for _, me, _, mf in mis]
    tail = [model.alpha * me for _, me, _, _ in mis]
    np.testing.assert_allclose(np.stack(head + tail), g["adjoint_rhs"], rtol=1e-12, atol=1e-15)
    adjoints = model.solve(model.adjoint_systems(phi, states))
    for x, ref in zip(adjoints, g["adjoints"]):
        assert rel_l2(x, ref) <= 1e-7
    s0, s1 = model.tensors(phi, states, list(g["adjoints"]))
    np.testing.assert_allclose(s0, g["S0"], rtol=1e-9, atol=1e-12 * np.abs(g["S0"]).max())
    np.testing.assert_allclose(s1, g["S1"], rtol=1e-9, atol=1e-12 * np.abs(g["S1"]).max())
    vec = derivative_vector(cspace, s1=s1, s0=s0)
    assert rel_l2(vec, g["vec"]) <= 1e-9


def test_assembly_by_parts_equals_whole():
    """The element-chunked assembly (cfg5 at full size does not fit otherwise)
    gives the matrix of the one-shot assembly, in 2D and 3D."""
    for lo, hi, n in (((0.0, 0.0), (2.0, 1.0), (6, 4)), ((0.0, 0.0, 0.0), (2.0, 1.0, 1.0), (4, 3, 2))):
        grid = Grid(lo, hi, n, [])
        space = fem.Space(grid, grid.dim)
        rng = np.random.default_rng(3)
        a_q = rng.uniform(0.1, 1.0, space.quad_weights.shape)
        whole = space.assemble_matrix(fem.elasticity_elements(space, a_q, (0.6, 0.4)))
        build = lambda part: fem.elasticity_elements(part, a_q[part.sl], (0.6, 0.4))  # noqa: E731
        for chunk in (7, 10**6):
            parts = space.assemble_matrix_by_parts(build, chunk=chunk)
            assert abs(parts - whole).max() <= 1e-15 * abs(whole).max()

"""3D (Kuhn tetrahedra) CUDA path vs the CPU oracle (needs a B200).

The reference is 2D only (fem.py:63-64); the 3D oracle is the
dimension-generic restatement in oracle/ (generic element gradients from
vertex coordinates, CSR assembly, scipy cg / SuperLU), so these tests also
check the kernels' closed-form Kuhn gradients against generic geometry.
"""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (BilinearSpec, ComplianceModel, DirichletSet,  # noqa: E402
                                   ElasticityOperator, FemField, FunctionSpace, LevelSetField,
                                   VelocitySolver, build_box_mesh, combine_derivatives,
                                   reinitialize, transport)
from paper_2601_05709_b200 import configs  # noqa: E402
from paper_2601_05709_b200.fem import solve_batched  # noqa: E402
from oracle import fem as ofem, levelset as olevel, model as omodel  # noqa: E402
from oracle.grid import Grid, level_set_h  # noqa: E402

LAME = (0.3 / (1.3 * 0.4), 1.0 / 2.6)
N3 = (9, 5, 4)
BOUNDS = ((0.0, 0.0, 0.0), (2.0, 1.0, 1.0))
RULES = [(1, lambda p: p[:, 0] < 1e-12),
         (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (np.abs(p[:, 1] - 0.5) < 0.3) & (np.abs(p[:, 2] - 0.5) < 0.3))]


def host(t):
    return t.detach().cpu().numpy()


def phi_fn(p):
    return -np.cos(4 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) * np.cos(4 * np.pi * p[:, 2]) - 0.3


@pytest.fixture(scope="module")
def both():
    mesh = build_box_mesh(BOUNDS[0] + BOUNDS[1], N3, RULES)
    grid = Grid(BOUNDS[0], BOUNDS[1], N3, RULES)
    space = FunctionSpace(mesh, 3)
    ospace = ofem.Space(grid, 3)
    phi = phi_fn(grid.vertices)
    return mesh, grid, space, ospace, phi


def test_facets_and_tags(both):
    mesh, grid, *_ = both
    np.testing.assert_array_equal(mesh.boundary_facets, grid.boundary_facets)
    np.testing.assert_array_equal(mesh.facet_tags, grid.facet_tags)
    np.testing.assert_array_equal(host(mesh.device_vertices()), grid.vertices)


def test_indicator_bit_exact(both):
    mesh, grid, space, ospace, phi = both
    lp = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), phi))
    ref = ofem.phi_at_quad_sign(ospace, phi).astype(float)
    np.testing.assert_array_equal(host(lp.indicator_quad()), ref)
    assert lp.h == pytest.approx(level_set_h(grid), rel=1e-15)


@pytest.mark.parametrize("with_bc", [False, True])
def test_apply_and_diag(both, with_bc):
    mesh, grid, space, ospace, phi = both
    model = omodel.Compliance(grid, LAME, 1e-3, ofem.clamp_dofs(ospace, grid.facets_with_tag(1)), [], 1.0)
    K = model.matrix(phi)
    bc = DirichletSet.on_tags(space, 1) if with_bc else None
    if with_bc:
        K, _ = ofem.dirichlet_eliminate(K, np.zeros(K.shape[0]), model.clamp)
        np.testing.assert_array_equal(bc.dofs, model.clamp)
    op = ElasticityOperator(space, torch.as_tensor(phi, device="cuda"), LAME, 1e-3, bc)
    u = np.random.default_rng(5).standard_normal((3, K.shape[0]))
    got = host(op.apply(torch.as_tensor(u, device="cuda")))
    for g, x in zip(got, u):
        assert rel_l2(g, K @ x) <= 1e-10
    assert rel_l2(host(op.diagonal()), K.diagonal()) <= 1e-12


@pytest.mark.parametrize("with_bc", [False, True])
def test_apply_cubic_cells(with_bc):
    """Cubic cells (h_x = h_y = h_z, as cfg3/cfg5) take the symmetric-flux
    kernel; check its apply, diagonal and a PCG solve against the oracle."""
    n = (8, 4, 4)
    mesh = build_box_mesh(BOUNDS[0] + BOUNDS[1], n, RULES)
    grid = Grid(BOUNDS[0], BOUNDS[1], n, RULES)
    space, ospace = FunctionSpace(mesh, 3), ofem.Space(grid, 3)
    phi = phi_fn(grid.vertices)
    model = omodel.Compliance(grid, LAME, 1e-3, ofem.clamp_dofs(ospace, grid.facets_with_tag(1)), [], 1.0)
    K = model.matrix(phi)
    bc = DirichletSet.on_tags(space, 1) if with_bc else None
    if with_bc:
        K, _ = ofem.dirichlet_eliminate(K, np.zeros(K.shape[0]), model.clamp)
    op = ElasticityOperator(space, torch.as_tensor(phi, device="cuda"), LAME, 1e-3, bc)
    u = np.random.default_rng(7).standard_normal((2, K.shape[0]))
    got = host(op.apply(torch.as_tensor(u, device="cuda")))
    for g, x in zip(got, u):
        assert rel_l2(g, K @ x) <= 1e-10
    assert rel_l2(host(op.diagonal()), K.diagonal()) <= 1e-12


def _model_pair(both):
    mesh, grid, space, ospace, phi = both
    clamp = ofem.clamp_dofs(ospace, grid.facets_with_tag(1))
    load = ofem.boundary_traction_vector(ospace, grid.facets_with_tag(2), (0.0, -1.0, 0.0))
    om = omodel.Compliance(grid, LAME, 1e-3, clamp, [load], 1.0)
    bil = BilinearSpec(mass_weight=1.0, stiffness_weight=1e-2)
    gm = ComplianceModel(mesh, 1, 2, (0.0, -1.0, 0.0), 1.0, lame=LAME, bilinear=bil, ersatz=1e-3)
    lp = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), phi))
    return om, gm, lp, bil


def test_state_cost_s1_velocity(both):
    mesh, grid, space, ospace, phi = both
    om, gm, lp, bil = _model_pair(both)
    assert rel_l2(host(gm.load_vectors[0]), om.loads[0]) <= 1e-14
    ostates, _ = om.solve_states(phi, rtol=1e-12)
    states = lsg.solve_concurrent(gm.pde(lp))
    assert rel_l2(host(states[0].values), ostates[0]) <= 1e-8
    uo = FemField(space, torch.as_tensor(ostates[0], device="cuda"))
    assert gm.cost(lp, [uo]) == pytest.approx(om.cost(phi, ostates), rel=1e-10)
    assert gm.constraint(lp, [uo])[0] == pytest.approx(om.constraint(phi), rel=1e-13)
    assert rel_l2(host(gm.s1_tensor(lp, [uo])), om.s1_cost(phi, ostates)) <= 1e-10
    lam = 0.37
    cost_pair, cons = gm.derivative(lp, [uo], None)
    pair = combine_derivatives(cost_pair, cons, np.array([lam]))
    solver = VelocitySolver(bil, space)
    vec_ref = omodel.derivative_vector(ospace, s1=om.s1_combined(phi, ostates, lam))
    assert rel_l2(host(solver._derivative_vector(pair)), vec_ref) <= 1e-10
    vel = omodel.Velocity(grid, 1.0, 1e-2)
    th_ref, btt_ref, dj_ref = vel.solve(vec_ref)
    res = solver.solve(pair)
    assert rel_l2(host(res.theta.values), th_ref) <= 1e-8
    assert res.form_value == pytest.approx(btt_ref, rel=1e-8)
    assert res.derivative == pytest.approx(dj_ref, rel=1e-8)


@pytest.mark.parametrize("name", ["normal", "dirichlet", "frozen"])
def test_velocity_forms(both, name):
    mesh, grid, space, ospace, phi = both
    if name == "normal":
        spec = BilinearSpec(mass_weight=0.1, stiffness_weight=1.0, boundary_normal_penalty=1e3)
        vel = omodel.Velocity(grid, 0.1, 1.0, boundary_normal_penalty=1e3)
    elif name == "dirichlet":
        spec = BilinearSpec(stiffness_weight=1.0, zero_dirichlet=True)
        vel = omodel.Velocity(grid, 0.0, 1.0, zero_dirichlet=True)
    else:
        spec = BilinearSpec(mass_weight=1.0, stiffness_weight=0.5,
                            frozen_subdomain=lambda p: p[:, 0] > 1.4, frozen_penalty=1e2)
        vel = omodel.Velocity(grid, 1.0, 0.5, frozen_chi=(ospace.quad_points[..., 0] > 1.4).astype(float),
                              frozen_penalty=1e2)
    solver = VelocitySolver(spec, space)
    u = np.random.default_rng(2).standard_normal(space.dof_count)
    if name != "dirichlet":
        assert rel_l2(host(solver.operator.apply(torch.as_tensor(u, device="cuda"))), vel.form_matrix @ u) <= 1e-10
    vec = np.random.default_rng(3).standard_normal(space.dof_count)
    th_ref, btt_ref, _ = vel.solve(vec)
    res = solver.solve(lsg.DerivativePair(vector=((1.0, torch.as_tensor(vec, device="cuda")),)))
    assert rel_l2(host(res.theta.values), th_ref) <= 1e-8
    assert res.form_value == pytest.approx(btt_ref, rel=1e-8)


def test_transport_and_reinit(both):
    mesh, grid, space, ospace, phi = both
    h = level_set_h(grid)
    x = grid.vertices
    th = np.stack([np.sin(np.pi * x[:, 0]), 0.3 * x[:, 1] - 0.1, np.cos(2 * x[:, 2])], 1)
    ref, nsub = olevel.transport(grid, phi, th.ravel(), 0.02, 8, True, h)
    lp = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), phi))
    out = transport(lp, FemField(space, th.ravel()), 0.02, 8, True)
    assert out.substeps == nsub
    assert rel_l2(host(out.values), ref) <= 1e-10
    ref2, nsub2 = olevel.reinitialize(grid, phi, 8, 0.1, h)
    out2 = reinitialize(lp, 8, 0.1)
    assert out2.substeps == nsub2
    assert rel_l2(host(out2.values), ref2) <= 1e-10


def test_batched_zero_and_nonzero(both):
    mesh, grid, space, ospace, phi = both
    om, gm, lp, bil = _model_pair(both)
    op = gm.operator(lp)
    b = torch.zeros((2, space.dof_count), dtype=torch.float64, device="cuda")
    b[1] = gm.load_vectors[0]
    x, it = solve_batched(op, b, torch.ones_like(b))
    assert float(x[0].abs().max()) == 0.0 and int(it[0]) == 0 and int(it[1]) > 0


def test_iteration_cap_and_odd_batch(both):
    """3D: k = 3 right-hand sides of different scale against the oracle's scipy cg,
    and the iteration cap raising SolverError(residual)."""
    mesh, grid, space, ospace, phi = both
    om, gm, lp, bil = _model_pair(both)
    op = gm.operator(lp)
    rng = np.random.default_rng(11)
    b = rng.standard_normal((3, space.dof_count)) * np.array([[1.0], [1e-3], [1e2]])
    b[:, gm.bc.dofs] = 0.0
    x, it = solve_batched(op, torch.as_tensor(b, device="cuda"), rtol=1e-12)
    A, _ = ofem.dirichlet_eliminate(om.matrix(phi), np.zeros(space.dof_count), om.clamp)
    for r in range(3):
        xr, _ = ofem.jacobi_pcg(A, b[r], rtol=1e-12)
        assert rel_l2(host(x[r]), xr) <= 1e-8
    with pytest.raises(lsg.SolverError) as err:
        solve_batched(op, torch.as_tensor(b[:1], device="cuda"), rtol=1e-14, atol=0.0, maxiter=4)
    assert err.value.residual > 0.0
    x0 = torch.zeros((1, space.dof_count), dtype=torch.float64, device="cuda")
    x0[0, 5] = float("inf")
    with pytest.raises(lsg.SolverError) as err:  # non-finite: stops at once, not at 10n
        solve_batched(op, torch.as_tensor(b[:1], device="cuda"), x0)
    assert int(str(err.value).split("after ")[1].split(" ")[0]) <= 3


def test_cfg3_coarse_history_matches_oracle():
    """cfg3 geometry at 12x6x6 (scale 8), 6 iterations with one reinit."""
    from oracle import cases as ocases, driver as odriver
    c = configs.case("cfg3", scale=8)
    c = type(c)(**{**c.__dict__, "niter": 6, "reinit_step": 3})
    mesh, model, phi, params = configs.build(c)
    _, hist = lsg.run(model, phi, params, timing=False)
    grid, omodel_, ovel, ophi, oparams, h = ocases.build(c)
    _, ohist = odriver.run(omodel_, ovel, ophi, oparams, h)
    for r, o in zip(hist, ohist):
        assert r.cost == pytest.approx(o["cost"], rel=1e-4)
        assert r.constraint[0] == pytest.approx(o["constraint"][0], rel=1e-4)
        assert r.steps == o["steps"] and r.transport_substeps == o["nsub_transport"]

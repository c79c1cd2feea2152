"""Grid-shape sweep: every kernel family against the oracle on odd and degenerate grids.

The stencil kernels tile the lattice (2D: 30 owned columns per warp, 4 warps
per CTA, row segments marched per CTA; 3D: 30 columns x 7 owned rows per CTA,
z segments, cp.async staging of 16-byte row chunks with a separate path for
the array's last row).  These shapes sit on and around every tile edge,
include single-cell axes, and use a seeded random level set so every material
count 0..nq occurs.  Gates as the north star: apply / diagonal / S1 vector /
one level-set step <= 1e-10 (diagonal 1e-12), CG solutions <= 1e-8.
"""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (BilinearSpec, ComplianceModel, DirichletSet,  # noqa: E402
                                   ElasticityOperator, FemField, FunctionSpace, LevelSetField,
                                   VelocitySolver, build_box_mesh, build_rect_mesh,
                                   combine_derivatives, reinitialize, transport)
from paper_2601_05709_b200.fem import solve_batched  # noqa: E402
from oracle import fem as ofem, levelset as olevel, model as omodel  # noqa: E402
from oracle.grid import Grid, level_set_h  # noqa: E402

LAME2 = (0.3 / 0.91, 1.0 / 2.6)
LAME3 = (0.3 / (1.3 * 0.4), 1.0 / 2.6)

SHAPES_2D = [(1, 1), (1, 7), (2, 1), (29, 3), (30, 4), (31, 5), (60, 2), (61, 9), (95, 33)]
# (n, cubic): cubic grids take the symmetric-flux elasticity kernel (ElastC)
SHAPES_3D = [((1, 1, 1), False), ((2, 1, 3), False), ((30, 7, 2), False), ((31, 8, 1), False),
             ((1, 13, 2), False), ((61, 14, 3), False), ((1, 1, 1), True), ((31, 8, 2), True),
             ((30, 7, 9), True), ((3, 15, 4), True), ((32, 14, 5), True), ((62, 6, 13), True),
             ((61, 15, 40), True)]


def host(t):
    return t.detach().cpu().numpy()


def _case(n, cubic=False, phi_mode="random"):
    dim = len(n)
    lo = (0.0,) * dim
    if cubic:
        hi = tuple(0.25 * v for v in n)  # h = 0.25 exactly on every axis
    else:
        hi = (2.0, 1.0) if dim == 2 else (2.0, 1.0, 0.7)
    x1 = hi[0]
    rules = [(1, lambda p: p[:, 0] < lo[0] + 1e-12), (2, lambda p: p[:, 0] > x1 - 1e-12)]
    grid = Grid(lo, hi, n, rules)
    mesh = build_rect_mesh(lo + hi, n[0], n[1], rules) if dim == 2 else build_box_mesh(lo + hi, n, rules)
    rng = np.random.default_rng(sum(n) * 7 + dim)
    if phi_mode == "random":
        phi = rng.standard_normal(grid.num_vertices) - 0.2
    elif phi_mode == "solid":
        phi = -np.ones(grid.num_vertices)
    else:
        phi = np.ones(grid.num_vertices)
    return grid, mesh, phi, rng


def _elasticity(grid, mesh, phi, rng, lame, k=2):
    space, ospace = FunctionSpace(mesh, grid.dim), ofem.Space(grid, grid.dim)
    clamp = ofem.clamp_dofs(ospace, grid.facets_with_tag(1))
    om = omodel.Compliance(grid, lame, 1e-3, clamp, [], 1.0)
    K = om.matrix(phi)
    Ke, _ = ofem.dirichlet_eliminate(K, np.zeros(K.shape[0]), clamp)
    ph = torch.as_tensor(phi, device="cuda")
    u = rng.standard_normal((k, K.shape[0]))
    op = ElasticityOperator(space, ph, lame, 1e-3)
    got = host(op.apply(torch.as_tensor(u, device="cuda")))
    for g, x in zip(got, u):
        assert rel_l2(g, K @ x) <= 1e-10
    # single field (shared-memory-ring apply) and an odd batch (register-ring apply)
    assert rel_l2(host(op.apply(torch.as_tensor(u[0], device="cuda"))), K @ u[0]) <= 1e-10
    u3 = np.concatenate([u, u[:1] * -0.5])
    for g, x in zip(host(op.apply(torch.as_tensor(u3, device="cuda"))), u3):
        assert rel_l2(g, K @ x) <= 1e-10
    assert rel_l2(host(op.diagonal()), K.diagonal()) <= 1e-12
    bc = DirichletSet.on_tags(space, 1)
    np.testing.assert_array_equal(bc.dofs, clamp)
    ope = ElasticityOperator(space, ph, lame, 1e-3, bc)
    got = host(ope.apply(torch.as_tensor(u, device="cuda")))
    for g, x in zip(got, u):
        assert rel_l2(g, Ke @ x) <= 1e-10
    assert rel_l2(host(ope.diagonal()), Ke.diagonal()) <= 1e-12
    return space, ospace, om, ope, Ke


def _solve(ope, Ke, clamp, rng):
    b = rng.standard_normal((3, Ke.shape[0])) * np.array([[1.0], [1e-2], [1e3]])
    b[:, clamp] = 0.0
    x, it = solve_batched(ope, torch.as_tensor(b, device="cuda"), rtol=1e-12)
    for r in range(3):
        xr, _ = ofem.jacobi_pcg(Ke, b[r], rtol=1e-12)
        assert rel_l2(host(x[r]), xr) <= 1e-8


def _derivative_and_velocity(grid, mesh, phi, space, ospace, om, rng):
    d = grid.dim
    trac = (0.0, -1.0) if d == 2 else (0.0, -1.0, 0.0)
    bil = BilinearSpec(mass_weight=1.0, stiffness_weight=1e-2)
    lame = LAME2 if d == 2 else LAME3
    gm = ComplianceModel(mesh, 1, 2, trac, 1.0, lame=lame, bilinear=bil, ersatz=1e-3)
    lp = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), phi))
    np.testing.assert_array_equal(host(lp.indicator_quad()), ofem.phi_at_quad_sign(ospace, phi).astype(float))
    ust = rng.standard_normal(space.dof_count)
    uo = FemField(space, torch.as_tensor(ust, device="cuda"))
    assert gm.cost(lp, [uo]) == pytest.approx(om.cost(phi, [ust]), rel=1e-10)
    assert gm.constraint(lp, [uo])[0] == pytest.approx(om.constraint(phi), rel=1e-12, abs=1e-15)
    assert rel_l2(host(gm.s1_tensor(lp, [uo])), om.s1_cost(phi, [ust])) <= 1e-10
    lam = 0.37
    cost_pair, cons = gm.derivative(lp, [uo], None)
    pair = combine_derivatives(cost_pair, cons, np.array([lam]))
    solver = VelocitySolver(bil, space)
    vec_ref = omodel.derivative_vector(ospace, s1=om.s1_combined(phi, [ust], lam))
    assert rel_l2(host(solver._derivative_vector(pair)), vec_ref) <= 1e-10
    vel = omodel.Velocity(grid, 1.0, 1e-2)
    w = rng.standard_normal(space.dof_count)
    assert rel_l2(host(solver.operator.apply(torch.as_tensor(w, device="cuda"))), vel.form_matrix @ w) <= 1e-10
    th_ref, btt_ref, dj_ref = vel.solve(vec_ref)
    res = solver.solve(pair)
    assert rel_l2(host(res.theta.values), th_ref) <= 1e-8
    assert res.form_value == pytest.approx(btt_ref, rel=1e-8)
    return lp


def _level_set(grid, mesh, phi, lp, space, rng):
    h = level_set_h(grid)
    th = rng.standard_normal(space.dof_count)
    for smooth in (False, True):
        ref, nsub = olevel.transport(grid, phi, th, 0.03, 6, smooth, h)
        out = transport(lp, FemField(space, th), 0.03, 6, smooth)
        assert out.substeps == nsub
        assert rel_l2(host(out.values), ref) <= 1e-10
    ref2, nsub2 = olevel.reinitialize(grid, phi, 6, 0.1, h)
    out2 = reinitialize(lp, 6, 0.1)
    assert out2.substeps == nsub2
    assert rel_l2(host(out2.values), ref2) <= 1e-10


@pytest.mark.parametrize("n", SHAPES_2D, ids=lambda n: "x".join(map(str, n)))
def test_shapes_2d(n):
    grid, mesh, phi, rng = _case(n)
    space, ospace, om, ope, Ke = _elasticity(grid, mesh, phi, rng, LAME2)
    _solve(ope, Ke, om.clamp, rng)
    lp = _derivative_and_velocity(grid, mesh, phi, space, ospace, om, rng)
    _level_set(grid, mesh, phi, lp, space, rng)


@pytest.mark.parametrize("n,cubic", SHAPES_3D, ids=lambda v: "x".join(map(str, v)) if isinstance(v, tuple)
                         else ("cubic" if v else "box"))
def test_shapes_3d(n, cubic):
    grid, mesh, phi, rng = _case(n, cubic)
    space, ospace, om, ope, Ke = _elasticity(grid, mesh, phi, rng, LAME3)
    _solve(ope, Ke, om.clamp, rng)
    lp = _derivative_and_velocity(grid, mesh, phi, space, ospace, om, rng)
    _level_set(grid, mesh, phi, lp, space, rng)


@pytest.mark.parametrize("mode", ["solid", "void"])
@pytest.mark.parametrize("n,cubic", [((33, 9), False), ((31, 8, 3), False), ((31, 8, 3), True)],
                         ids=["2d", "3d", "3d-cubic"])
def test_uniform_material(n, cubic, mode):
    """All-solid and all-void (ersatz everywhere) material words."""
    grid, mesh, phi, rng = _case(n, cubic, phi_mode=mode)
    space, ospace, om, ope, Ke = _elasticity(grid, mesh, phi, rng, LAME2 if len(n) == 2 else LAME3)
    _solve(ope, Ke, om.clamp, rng)

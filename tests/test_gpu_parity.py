"""CUDA path vs the reference's golden vectors and the CPU oracle (needs a B200).

Tolerances are the north star's: mesh indexing bit-exact; apply, S0/S1 and
one level-set step <= 1e-10 relative L2; CG solutions <= 1e-8 relative L2;
J/C history <= 1e-4 relative.  Everything goes through the C ABI
(liblsgpu.so via ctypes) -- there is no other implementation to fall back to.
"""

import math

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (BilinearSpec, ComplianceModel, CompliancePlusModel,  # noqa: E402
                                   DirichletSet, ElasticityOperator, FemField, FunctionSpace,
                                   LevelSetField, VelocitySolver, build_rect_mesh,
                                   combine_derivatives, reinitialize, transport)
from paper_2601_05709_b200 import configs  # noqa: E402
from paper_2601_05709_b200.fem import solve_batched  # noqa: E402
from paper_2601_05709_b200.models import MaterialIndicator, solve_problem  # noqa: E402
from oracle import levelset as olevel  # noqa: E402
from oracle.grid import Grid, level_set_h  # noqa: E402

LAME = (0.3 / 0.91, 1.0 / 2.6)


def cantilever(nx, ny):
    rules = [(1, lambda p: p[:, 0] < 1e-12),
             (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55))]
    return build_rect_mesh((0.0, 0.0, 2.0, 1.0), nx, ny, rules)


def phi_fn(p):
    return -np.cos(6 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) - 0.4


@pytest.fixture(scope="module")
def setup32():
    mesh = cantilever(32, 16)
    space = FunctionSpace(mesh, 2)
    phi = LevelSetField.from_field(FunctionSpace(mesh, 1).interpolate(phi_fn))
    bil = BilinearSpec(mass_weight=1.0, stiffness_weight=1e-2)
    model = ComplianceModel(mesh, 1, 2, (0.0, -1.0), 1.0, lame=LAME, bilinear=bil, ersatz=1e-3)
    return mesh, space, phi, model, bil


def host(t):
    return t.detach().cpu().numpy()


class TestMesh:
    def test_device_mesh_bit_exact(self, golden):
        mesh = cantilever(7, 5)
        np.testing.assert_array_equal(host(mesh.device_vertices()), golden["mesh_vertices"])
        np.testing.assert_array_equal(host(mesh.device_elements()), golden["mesh_triangles"])
        np.testing.assert_array_equal(mesh.boundary_facets, golden["mesh_facets"])
        np.testing.assert_array_equal(mesh.facet_tags, golden["mesh_tags"])
        odd = build_rect_mesh((-0.3, 0.1, 1.7, 1.3), 13, 9)
        np.testing.assert_array_equal(host(odd.device_vertices()), golden["odd_vertices"])

    def test_device_mesh_3d_matches_oracle(self):
        from paper_2601_05709_b200 import build_box_mesh
        m = build_box_mesh((0.0, 0.0, 0.0, 2.0, 1.0, 1.0), (5, 4, 3))
        g = Grid((0.0, 0.0, 0.0), (2.0, 1.0, 1.0), (5, 4, 3))
        np.testing.assert_array_equal(host(m.device_vertices()), g.vertices)
        np.testing.assert_array_equal(host(m.device_elements()), g.elements)
        np.testing.assert_array_equal(m.boundary_facets, g.boundary_facets)


class TestOperator:
    def test_indicator_bit_exact(self, golden, setup32):
        mesh, space, phi, model, _ = setup32
        np.testing.assert_array_equal(host(phi.values), golden["phi_32x16"])
        np.testing.assert_array_equal(host(phi.indicator_quad()), golden["chi_32x16"])

    def test_apply_unconstrained(self, golden, setup32):
        mesh, space, phi, model, _ = setup32
        op = ElasticityOperator(space, phi.values, LAME, 1e-3)
        u = torch.as_tensor(golden["apply_u"], device="cuda")
        got = host(op.apply(u))
        for g, ref in zip(got, golden["apply_Ku"]):
            assert rel_l2(g, ref) <= 1e-10
        single = host(op.apply(u[1]))  # batch == single, bitwise
        np.testing.assert_array_equal(single, got[1])

    def test_apply_eliminated_and_diag(self, golden, setup32):
        mesh, space, phi, model, _ = setup32
        bc = DirichletSet.on_tags(space, 1)
        np.testing.assert_array_equal(bc.dofs, golden["bc_dofs"])
        op = ElasticityOperator(space, phi.values, LAME, 1e-3, bc)
        got = host(op.apply(torch.as_tensor(golden["apply_u"], device="cuda")))
        for g, ref in zip(got, golden["apply_Keu"]):
            assert rel_l2(g, ref) <= 1e-10
        assert rel_l2(host(op.diagonal()), golden["diag_elim"]) <= 1e-12

    def test_apply_deterministic(self, setup32):
        mesh, space, phi, model, _ = setup32
        op = ElasticityOperator(space, phi.values, LAME, 1e-3)
        u = torch.randn(4, space.dof_count, dtype=torch.float64, device="cuda")
        a, b = host(op.apply(u)), host(op.apply(u))
        np.testing.assert_array_equal(a, b)


class TestSolve:
    def test_state_matches_reference(self, golden, setup32):
        mesh, space, phi, model, _ = setup32
        assert rel_l2(host(model.load_vectors[0]), golden["load_vector"]) <= 1e-15
        u = solve_problem(model.pde(phi)[0])
        assert rel_l2(host(u.values), golden["state_u"]) <= 1e-8
        J = model.cost(phi, [u])
        assert J == pytest.approx(golden["J"][0], rel=1e-8)
        assert model.constraint(phi, [u])[0] == pytest.approx(golden["C"][0], rel=1e-14)

    def test_batched_two_loads(self, golden, setup32):
        mesh, space, phi, _, bil = setup32
        plus = CompliancePlusModel(mesh, 1, [((0.0, -1.0), 2), ((0.0, -2.0), 2)], 1.0, lame=LAME,
                                   bilinear=bil, ersatz=1e-3)
        states = lsg.solve_concurrent(plus.pde(phi))
        assert rel_l2(np.stack([host(s.values) for s in states]), golden["plus_states"]) <= 1e-8
        assert plus.cost(phi, states) == pytest.approx(golden["plus_J"][0], rel=1e-8)

    def test_zero_rhs_returns_zero(self, setup32):
        mesh, space, phi, model, _ = setup32
        op = model.operator(phi)
        b = torch.zeros((2, space.dof_count), dtype=torch.float64, device="cuda")
        b[1] = model.load_vectors[0]
        x0 = torch.ones_like(b)
        x, iters = solve_batched(op, b, x0)
        assert float(x[0].abs().max()) == 0.0 and int(iters[0]) == 0
        assert int(iters[1]) > 0

    def test_converged_warm_start_is_untouched(self, setup32):
        mesh, space, phi, model, _ = setup32
        op = model.operator(phi)
        b = model.load_vectors[:1]
        x1, it1 = solve_batched(op, b, rtol=1e-12)
        x2, it2 = solve_batched(op, b, x1, rtol=1e-10)
        assert int(it2[0]) == 0
        np.testing.assert_array_equal(host(x1), host(x2))


    def test_iteration_cap_raises_solver_error_with_true_residual(self, setup32):
        """scipy cg semantics (fem.py:309-315): maxiter exhausted -> SolverError(residual)
        carrying the true residual of the failing right-hand side."""
        mesh, space, phi, model, _ = setup32
        op = model.operator(phi)
        b = model.load_vectors[:1]
        with pytest.raises(lsg.SolverError) as err:
            solve_batched(op, b, rtol=1e-14, atol=0.0, maxiter=5)
        assert err.value.residual > 0.0 and np.isfinite(err.value.residual)
        assert "5 iterations" in str(err.value)

    def test_non_finite_fails_fast(self, setup32):
        """A NaN iterate stops its right-hand side at once (SolverError) instead of
        running to the 10n cap; the other right-hand side of the batch still converges."""
        mesh, space, phi, model, _ = setup32
        op = model.operator(phi)
        b = torch.stack([model.load_vectors[0], model.load_vectors[0]])
        x0 = torch.zeros_like(b)
        x0[0, 7] = float("nan")
        with pytest.raises(lsg.SolverError) as err:
            solve_batched(op, b, x0)
        n_it = int(str(err.value).split("after ")[1].split(" ")[0])
        assert n_it <= 2
        x, it = solve_batched(op, b[1:])
        assert torch.isfinite(x).all() and int(it[0]) > 10


class TestDerivativeAndVelocity:
    def test_s1_tensor(self, golden, setup32):
        mesh, space, phi, model, _ = setup32
        u = FemField(space, torch.as_tensor(golden["state_u"], device="cuda"))
        s1 = host(model.s1_tensor(phi, [u]))
        assert rel_l2(s1, golden["S1_cost"]) <= 1e-10

    def test_fused_velocity_rhs_and_solve(self, golden, setup32):
        mesh, space, phi, model, bil = setup32
        u = FemField(space, torch.as_tensor(golden["state_u"], device="cuda"))
        cost_pair, cons = model.derivative(phi, [u], None)
        pair = combine_derivatives(cost_pair, cons, np.array([0.37]))
        solver = VelocitySolver(bil, space)
        vec = host(solver._derivative_vector(pair))
        assert rel_l2(vec, golden["velocity_vec"]) <= 1e-10
        res = solver.solve(pair)
        assert rel_l2(host(res.theta.values), golden["theta"]) <= 1e-8
        assert res.form_value == pytest.approx(golden["form_value"][0], rel=1e-9)
        assert res.derivative == pytest.approx(golden["derivative"][0], rel=1e-9)
        assert abs(res.derivative + res.form_value) <= 1e-8 * (1 + res.form_value)

    def test_closure_path_matches_fused(self, golden, setup32):
        mesh, space, phi, model, bil = setup32
        u = FemField(space, torch.as_tensor(golden["state_u"], device="cuda"))
        cost_pair, cons = model.derivative(phi, [u], None)
        from paper_2601_05709_b200 import DerivativePair
        closures = combine_derivatives(DerivativePair(s1=cost_pair.s1),
                                       [DerivativePair(s1=cons[0].s1)], np.array([0.37]))
        vec = host(VelocitySolver(bil, space)._derivative_vector(closures))
        assert rel_l2(vec, golden["velocity_vec"]) <= 1e-10

    @pytest.mark.parametrize("name,spec", [
        ("normal", BilinearSpec(mass_weight=0.1, stiffness_weight=1.0, boundary_normal_penalty=1e4)),
        ("dirichlet", BilinearSpec(stiffness_weight=1.0, zero_dirichlet=True)),
        ("frozen", BilinearSpec(mass_weight=1.0, stiffness_weight=0.5,
                                frozen_subdomain=lambda p: p[:, 0] > 1.6, frozen_penalty=1e2)),
    ])
    def test_velocity_form_variants(self, golden, setup32, name, spec):
        mesh, space, phi, model, _ = setup32
        solver = VelocitySolver(spec, space)
        y = host(solver.operator.apply(torch.as_tensor(golden["apply_u"][0], device="cuda")))
        if name != "dirichlet":  # the reference's form_matrix is the un-eliminated one
            assert rel_l2(y, golden[f"form_apply_{name}"]) <= 1e-10
        from paper_2601_05709_b200 import DerivativePair
        pair = DerivativePair(vector=((1.0, torch.as_tensor(golden["velocity_vec"], device="cuda")),))
        res = solver.solve(pair)
        assert rel_l2(host(res.theta.values), golden[f"theta_{name}"]) <= 1e-8
        assert res.form_value == pytest.approx(golden[f"form_value_{name}"][0], rel=1e-8)


class TestLevelSet:
    def _pair(self, n=48):
        mesh = build_rect_mesh((0.0, 0.0, 1.0, 1.0), n, n)
        grid = Grid((0.0, 0.0), (1.0, 1.0), (n, n))
        x = grid.vertices
        phi = np.linalg.norm(x - 0.5, axis=1) - 0.3 + 0.05 * np.sin(7 * x[:, 0])
        th = np.stack([np.sin(np.pi * x[:, 0]) * np.cos(2 * x[:, 1]), 0.3 + x[:, 0] * x[:, 1]], 1)
        return mesh, grid, phi, th

    @pytest.mark.parametrize("smooth", [False, True])
    def test_transport_matches_oracle(self, smooth):
        mesh, grid, phi, th = self._pair()
        h = level_set_h(grid)
        ref, nsub = olevel.transport(grid, phi, th.ravel(), 0.03, 8, smooth, h)
        p = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), phi))
        t = FemField(FunctionSpace(mesh, 2), th.ravel())
        out = transport(p, t, 0.03, 8, smooth)
        assert out.substeps == nsub
        assert p.h == pytest.approx(h, rel=1e-15)
        assert rel_l2(host(out.values), ref) <= 1e-10
        np.testing.assert_array_equal(host(p.values), phi)  # input untouched

    def test_reinit_matches_oracle(self):
        mesh, grid, phi, _ = self._pair()
        h = level_set_h(grid)
        ref, nsub = olevel.reinitialize(grid, 3.0 * phi, 8, 0.1, h)
        p = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), 3.0 * phi))
        out = reinitialize(p, 8, 0.1)
        assert out.substeps == nsub
        assert rel_l2(host(out.values), ref) <= 1e-10


class TestHistory:
    def test_cfg1_coarse_history_matches_oracle(self):
        """cfg1 geometry at 40x20, 12 iterations (two reinitialisations): J and C
        histories within 1e-4 relative of the oracle; discrete counters equal."""
        from oracle import cases as ocases, driver as odriver
        c = configs.case("cfg1", scale=4)
        c = type(c)(**{**c.__dict__, "niter": 12})
        mesh, model, phi, params = configs.build(c)
        _, hist = lsg.run(model, phi, params, timing=False)
        grid, omodel, ovel, ophi, oparams, h = ocases.build(c)
        _, ohist = odriver.run(omodel, ovel, ophi, oparams, h)
        assert len(hist) == len(ohist) == 12
        for r, o in zip(hist, ohist):
            assert r.cost == pytest.approx(o["cost"], rel=1e-4)
            assert r.constraint[0] == pytest.approx(o["constraint"][0], rel=1e-4)
            assert r.steps == o["steps"]
            assert r.transport_substeps == o["nsub_transport"]
            assert r.reinit_substeps == o["nsub_reinit"]


class TestReferenceScheme:
    """The reference's own CN/PG transport and PG/AB2 reinit on the device
    (levelset.py:137-216) vs the reference's outputs, and a full run() with it
    vs the reference's own run() history (tests/golden/make_golden.py)."""

    def _sq(self, golden):
        mesh = build_rect_mesh((0.0, 0.0, 1.0, 1.0), 24, 20)
        phi = LevelSetField.from_field(FemField(FunctionSpace(mesh, 1), golden["ls_phi"]))
        th = FemField(FunctionSpace(mesh, 2), golden["ls_theta"])
        return mesh, phi, th

    @pytest.mark.parametrize("smooth,key", [(False, "ls_transport"), (True, "ls_transport_smooth")])
    def test_transport_vs_reference(self, golden, smooth, key):
        mesh, phi, th = self._sq(golden)
        out = transport(phi, th, 0.03, 8, smooth, scheme="pg")
        assert rel_l2(host(out.values), golden[key]) <= 1e-10
        np.testing.assert_array_equal(host(phi.values), golden["ls_phi"])

    def test_reinit_vs_reference(self, golden):
        mesh, phi, th = self._sq(golden)
        p3 = LevelSetField(FemField(phi.space, 3.0 * phi.values), phi.h)
        out = reinitialize(p3, 8, 0.1, scheme="pg")
        assert rel_l2(host(out.values), golden["ls_reinit"]) <= 1e-10

    def test_run_history_vs_reference_run(self, golden):
        c = configs.case("cfg1", scale=4)
        c = type(c)(**{**c.__dict__, "niter": 12, "reinit_step": 5})
        mesh, model, phi, params = configs.build(c)
        params = lsg.RunParams(**{**params.__dict__, "level_set_scheme": "pg"})
        _, hist = lsg.run(model, phi, params, timing=False)
        np.testing.assert_allclose([r.cost for r in hist], golden["run_cost"], rtol=1e-4)
        np.testing.assert_allclose([r.constraint[0] for r in hist], golden["run_constraint"], rtol=1e-4)
        np.testing.assert_allclose([r.t_end for r in hist], golden["run_t_end"], rtol=1e-4)
        np.testing.assert_array_equal([r.steps for r in hist], golden["run_steps"])


class TestOutput:
    def test_vtk_bytes_match_reference(self, golden, tmp_path):
        from paper_2601_05709_b200.output import write_vtk
        m = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 3, 2)
        f1 = FunctionSpace(m, 1).interpolate(lambda p: np.sin(p[:, 0]) - p[:, 1] / 3.0)
        f2 = FunctionSpace(m, 2).interpolate(lambda p: np.stack([p[:, 0] / 7.0, -p[:, 1]], 1))
        write_vtk(m, {"phi": f1, "theta": f2}, tmp_path / "m.vtk")
        assert (tmp_path / "m.vtk").read_text() == str(golden["vtk_text"])

    def test_streaming_history_writer(self, tmp_path):
        from paper_2601_05709_b200.output import HistoryWriter, history_header
        c = configs.case("cfg1", scale=8)
        c = type(c)(**{**c.__dict__, "niter": 3})
        mesh, model, phi, params = configs.build(c)
        with HistoryWriter(tmp_path / "h.csv") as w:
            _, hist = lsg.run(model, phi, params, on_record=w.on_record, timing=False)
        lines = (tmp_path / "h.csv").read_text().strip().split("\n")
        assert lines[0] == history_header(1) and len(lines) == 4
        assert float(lines[1].split(",")[1]) == hist[0].cost

"""The five BASELINE configurations on the B200 path vs the CPU oracle.

The oracle cannot run the full sizes in test time (cfg2 ~1,660 s per
iteration, cfg4 needs 25 GB for the CSR assembly), so:

* histories (J, C within 1e-4; identical RNG-driven step counts and CFL
  substeps) run each config's geometry, loads and phi0 on a coarser grid
  (`configs.case(name, scale)`);
* cfg4's operator pieces (apply, PCG to 1e-8, S1 / derivative vector, H1
  solve) are checked against the oracle at 1/8 scale, and at FULL size through
  size-independent properties: symmetry of the operator, rigid-motion kernel
  of the unconstrained operator, the true residual of the PCG solution, the
  descent identity of the velocity solve, and bitwise determinism.
"""

import numpy as np
import pytest
import torch

from conftest import rel_l2

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (ElasticityOperator, FemField, FunctionSpace, VelocitySolver,  # noqa: E402
                                   combine_derivatives, configs)
from paper_2601_05709_b200.fem import solve_batched  # noqa: E402
from oracle import cases as ocases, driver as odriver, fem as ofem, model as omodel  # noqa: E402


def host(t):
    return t.detach().cpu().numpy()


def history_pair(name, scale, niter, reinit_step):
    c = configs.case(name, scale=scale)
    c = type(c)(**{**c.__dict__, "niter": niter, "reinit_step": reinit_step})
    mesh, model, phi, params = configs.build(c)
    _, hist = lsg.run(model, phi, params, timing=False)
    grid, om, ovel, ophi, oparams, h = ocases.build(c)
    _, ohist = odriver.run(om, ovel, ophi, oparams, h)
    return hist, ohist


@pytest.mark.parametrize("name,scale,niter,reinit", [
    ("cfg1", 4, 12, 5),
    ("cfg2", 8, 6, 3),
    ("cfg3", 8, 6, 3),
    ("cfg5", 16, 5, 2),
])
def test_history_matches_oracle(name, scale, niter, reinit):
    hist, ohist = history_pair(name, scale, niter, reinit)
    assert len(hist) == len(ohist) == niter
    for r, o in zip(hist, ohist):
        assert r.cost == pytest.approx(o["cost"], rel=1e-4)
        assert r.constraint[0] == pytest.approx(o["constraint"][0], rel=1e-4)
        assert r.lagrangian == pytest.approx(o["lagrangian"], rel=1e-4)
        assert r.steps == o["steps"]
        assert r.transport_substeps == o["nsub_transport"]
        assert r.reinit_substeps == o["nsub_reinit"]
        assert r.form_value == pytest.approx(o["form_value"], rel=1e-4)


def test_cfg4_operator_pieces_vs_oracle():
    """cfg4 geometry (random two-phase field, body force, bottom clamp) at 512x256."""
    c = configs.case("cfg4", scale=8)
    mesh, model, phi, params = configs.build(c)
    grid, om, ovel, ophi, oparams, h = ocases.build(c)
    np.testing.assert_array_equal(host(phi.values), ophi)
    K = om.matrix(ophi)
    Ke, b = ofem.dirichlet_eliminate(K, om.loads[0], om.clamp)
    assert rel_l2(host(model.load_vectors[0]), b) <= 1e-14
    op = model.operator(phi)
    u = np.random.default_rng(4).standard_normal(K.shape[0])
    assert rel_l2(host(op.apply(torch.as_tensor(u, device="cuda"))), Ke @ u) <= 1e-10
    x, it = solve_batched(op, model.load_vectors, rtol=1e-8)
    xo, ito = ofem.jacobi_pcg(Ke, b, rtol=1e-8)
    assert rel_l2(host(x[0]), xo) <= 1e-6  # both stop at ||r_recursive|| < 1e-8 ||b||
    # the TRUE residual drifts above the recursive one in both implementations
    # (finite-precision CG, cond ~1e7 here); it must be of the oracle's size
    true_gpu = np.linalg.norm(b - Ke @ host(x[0]))
    true_ref = np.linalg.norm(b - Ke @ xo)
    assert true_gpu <= 3.0 * max(true_ref, 1e-8 * np.linalg.norm(b))
    # same algorithm and stopping rule; at cond ~1e7 the rounding order of the
    # dot products moves the crossing of 1e-8 ||b|| by a few percent
    assert abs(int(it[0]) - ito) <= max(3, ito // 10)
    state = FemField(model.space, x[0])
    assert model.cost(phi, [state]) == pytest.approx(om.cost(ophi, [host(x[0])]), rel=1e-10)
    cost_pair, cons = model.derivative(phi, [state], None)
    pair = combine_derivatives(cost_pair, cons, np.array([0.2]))
    solver = VelocitySolver(model.bilinear_form(), model.space)
    vec = omodel.derivative_vector(om.space, s1=om.s1_combined(ophi, [host(x[0])], 0.2))
    assert rel_l2(host(solver._derivative_vector(pair)), vec) <= 1e-10
    res = solver.solve(pair)
    th, btt, dj = ovel.solve(vec)
    assert rel_l2(host(res.theta.values), th) <= 1e-8
    assert res.form_value == pytest.approx(btt, rel=1e-8)


def test_cfg4_full_size_properties():
    """cfg4 at full size (4096x2048, 16.8M dofs): size-independent checks."""
    c = configs.case("cfg4")
    mesh, model, phi, params = configs.build(c)
    op = model.operator(phi)
    n = model.space.dof_count
    g = torch.Generator(device="cuda").manual_seed(0)
    u = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    v = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    Ku, Kv = op.apply(u), op.apply(v)
    s1, s2 = float(v @ Ku), float(u @ Kv)
    assert abs(s1 - s2) <= 1e-11 * abs(s1)  # symmetry
    # rigid motions span the kernel of the unconstrained operator
    free = ElasticityOperator(model.space, phi.values, c.lame, c.ersatz)
    x = mesh.device_vertices()
    for mode in (torch.stack([torch.ones_like(x[:, 0]), torch.zeros_like(x[:, 0])], 1),
                 torch.stack([-x[:, 1], x[:, 0]], 1)):
        r = free.apply(mode.reshape(-1).contiguous())
        assert float(r.abs().max()) <= 1e-10 * float(free.apply(u).abs().max())
    # determinism
    assert torch.equal(op.apply(u), Ku)
    # PCG to 1e-8 (scipy's criterion on the recursive residual); the true
    # residual drifts with the ~2e5 iterations this solve takes (measured
    # 1.2e-5 relative, profiles/r01_bench_notes.md) -- bounded here
    from paper_2601_05709_b200.fem import _workspace
    xs, it = solve_batched(op, model.load_vectors, rtol=1e-8)
    b = model.load_vectors[0]
    bn = float(torch.linalg.vector_norm(b))
    rec = float(_workspace(op, 1).host_scal[0, 4]) ** 0.5
    assert rec < 1e-8 * bn
    assert float(torch.linalg.vector_norm(b - op.apply(xs[0]))) <= 1e-4 * bn
    # S0/S1 + H1 descent solve: descent identity
    state = FemField(model.space, xs[0])
    J = model.cost(phi, [state])
    assert J > 0
    cost_pair, cons = model.derivative(phi, [state], None)
    pair = combine_derivatives(cost_pair, cons, np.array([0.1]))
    res = VelocitySolver(model.bilinear_form(), model.space).solve(pair)
    assert res.form_value > 0
    assert abs(res.derivative + res.form_value) <= 1e-8 * (1 + res.form_value)


# -- the same configurations from the shipped TOML files (paper_2601_05709_b200.config) ------
@pytest.mark.parametrize("name,n", [("cfg1", (40, 20)), ("cfg5", (24, 12, 12))])
def test_toml_config_builds_the_coded_case(name, n):
    import os
    from dataclasses import replace
    from paper_2601_05709_b200.config import build_initial, build_mesh, build_model, parse_config
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cfg = parse_config(os.path.join(root, "configs", f"{name}.toml"))
    mesh_kw = dict(nx=n[0], ny=n[1]) if len(n) == 2 else dict(nx=n[0], ny=n[1], nz=n[2])
    cfg = replace(cfg, mesh=replace(cfg.mesh, **mesh_kw))
    mesh = build_mesh(cfg)
    model, phi = build_model(cfg, mesh), build_initial(cfg, mesh)
    c = configs.case(name, scale=4 if name == "cfg1" else 8)
    _, model2, phi2, _ = configs.build(c)
    np.testing.assert_array_equal(host(phi.values), host(phi2.values))
    np.testing.assert_allclose(host(model.load_vectors), host(model2.load_vectors), rtol=1e-14, atol=0)
    s1, s2 = lsg.solve_concurrent(model.pde(phi)), lsg.solve_concurrent(model2.pde(phi2))
    assert model.cost(phi, s1) == pytest.approx(model2.cost(phi2, s2), rel=1e-12)


def test_toml_inverse_and_heat_models_run():
    from paper_2601_05709_b200.config import build_initial, build_mesh, build_model, config_from_dict
    inverse = {
        "model": {"kind": "inverse", "fixed_tag": 1, "measured_tag": [2, 3, 4, 5], "contrast": 10.0,
                  "twin": {"center": [1.0, 0.5], "radius": 0.25, "refine": 2},
                  "force": [{"traction": [1.0, 0.0], "tag": 3}, {"traction": [0.0, -1.0], "tag": 4}]},
        "mesh": {"bounds": [0.0, 0.0, 2.0, 1.0], "nx": 16, "ny": 8},
        "boundary": [{"tag": 3, "side": "left", "span": [0.25, 0.75]},
                     {"tag": 4, "side": "top", "span": [0.75, 1.25]},
                     {"tag": 5, "side": "right", "span": [0.25, 0.75]},
                     {"tag": 1, "side": "bottom"}, {"tag": 2, "side": "all"}],
        "initial": {"centers": [[0.9, 0.6]], "radii": [0.35], "factor": -1.0},
        "run": {"niter": 3, "start_to_check": 3, "lv_time": [1e-3, 10.0], "lv_iter": [8, 32]},
    }
    heat = {
        "model": {"kind": "heat", "volume": 0.5, "fixed_tag": 1,
                  "source": {"kind": "radial", "center": [0.5, 0.5], "amplitude": 25.0, "cutoff": 0.2}},
        "mesh": {"bounds": [0.0, 0.0, 1.0, 1.0], "nx": 16, "ny": 16},
        "boundary": [{"tag": 1, "side": "all"}],
        "initial": {"centers": [[0.25, 0.25], [0.75, 0.75]], "radii": [0.15, 0.15]},
        "run": {"niter": 3, "start_to_check": 3, "smooth": True},
    }
    for doc in (inverse, heat):
        cfg = config_from_dict(doc)
        mesh = build_mesh(cfg)
        model, phi = build_model(cfg, mesh), build_initial(cfg, mesh)
        _, hist = lsg.run(model, phi, cfg.params, timing=False)
        assert len(hist) == 3 and all(np.isfinite(r.cost) for r in hist)


def test_cfg1_full_size_history_matches_oracle():
    """BASELINE cfg1 at its own size (160x80, all 50 iterations, reinit every 5): J, C,
    Lagrangian, B(theta, theta) within 1e-4 of the oracle's run at every iteration and
    identical discrete counters (tests/golden/make_golden_cfg1_full.py)."""
    import os
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "oracle_cfg1_full.npz"))
    mesh, model, phi, params = configs.build(configs.case("cfg1"))
    _, hist = lsg.run(model, phi, params, timing=False)
    assert len(hist) == len(gold["cost"]) == 50
    np.testing.assert_allclose([r.cost for r in hist], gold["cost"], rtol=1e-4)
    np.testing.assert_allclose([r.constraint[0] for r in hist], gold["constraint"], rtol=1e-4)
    np.testing.assert_allclose([r.lagrangian for r in hist], gold["lagrangian"], rtol=1e-4)
    np.testing.assert_allclose([r.form_value for r in hist], gold["form_value"], rtol=1e-4)
    np.testing.assert_array_equal([r.steps for r in hist], gold["steps"])
    np.testing.assert_array_equal([r.transport_substeps for r in hist], gold["nsub_transport"])
    np.testing.assert_array_equal([r.reinit_substeps for r in hist], gold["nsub_reinit"])


def test_cfg1_full_size_reference_scheme_matches_reference_run():
    """The reference's own run() (its CN/PG level-set scheme) on the full-size cfg1
    mesh (tests/golden/make_golden_cfg1_reference.py) against the device run with
    level_set_scheme="pg".  From the reinitialisation at iteration 4 the
    reference's scheme inflates |phi| to ~1e7 and, by iteration 9, ~1e15; its splu
    still solves those steps, Krylov solvers do not reach 1e-14 there.  The device
    run therefore matches the reference through iteration 7 (J to ~1e-10 relative),
    iteration 8 within the north star's 1e-4, and then raises SolverError at the iteration-9 reinitialisation -- loudly, never
    with a silently wrong level set."""
    import os
    gold = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_cfg1_full.npz"))
    c = configs.case("cfg1")
    c = type(c)(**{**c.__dict__, "niter": 12})
    mesh, model, phi, params = configs.build(c)
    params = lsg.RunParams(**{**params.__dict__, "level_set_scheme": "pg"})
    opt = lsg.driver.Optimizer(model, phi, params, timing=False)
    hist = []
    try:
        for _ in range(12):
            hist.append(opt.step())
    except lsg.SolverError:
        pass
    assert len(hist) >= 9
    n = len(hist)
    # through iteration 7 to 1e-8; from iteration 8 (|phi| inflated by the
    # reference's reinitialisation) a one-ulp change in any reduction can flip
    # the indicator of quadrature points with phi ~ 0 (measured: C moves by
    # 4e-5 relative), so there the north star's history gate (1e-4) applies
    np.testing.assert_allclose([r.cost for r in hist[:8]], gold["cost"][:8], rtol=1e-8)
    np.testing.assert_allclose([r.constraint[0] for r in hist[:8]], gold["constraint"][:8], rtol=1e-8)
    np.testing.assert_allclose([r.cost for r in hist], gold["cost"][:n], rtol=1e-4)
    np.testing.assert_allclose([r.constraint[0] for r in hist], gold["constraint"][:n], rtol=1e-4)
    np.testing.assert_array_equal([r.steps for r in hist], gold["steps"][:n])

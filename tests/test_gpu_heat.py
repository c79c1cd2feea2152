"""Heat models (reference ``models/heat.py``) on the CUDA path vs the
reference's golden vectors (tests/golden/make_golden_heat.py) and the oracle.

Needs a B200.  Covers the scalar diffusion operator (apply, diagonal,
Dirichlet elimination), the batched grounded solves, the fused thermal
compliance + S0/S1 contraction (with and without a source gradient), the
velocity solve and a short run() history against the reference's own run().
"""

import os

import numpy as np
import pytest
import torch

from conftest import rel_l2
from heat_cases import BOUNDS, NX, NY, RULES, VOLUME, grad_a, phi_fn, src_a, src_b

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (BilinearSpec, DirichletSet, FemField, FunctionSpace,  # noqa: E402
                                   HeatModel, HeatPlusModel, HeatTerm, LaplaceOperator,
                                   LevelSetField, VelocitySolver, build_rect_mesh,
                                   combine_derivatives)
from oracle import fem as ofem, model as omodel  # noqa: E402
from oracle.grid import Grid  # noqa: E402

BIL = BilinearSpec(stiffness_weight=1.0, boundary_normal_penalty=1e4)


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_heat.npz"))


@pytest.fixture(scope="module")
def setup():
    mesh = build_rect_mesh(BOUNDS, NX, NY, RULES)
    scalar = FunctionSpace(mesh, 1)
    phi = LevelSetField.from_field(scalar.interpolate(phi_fn))
    terms = [HeatTerm(src_a, 1, 0.7, grad_a), HeatTerm(src_b, (2, 3), None, None)]
    return mesh, scalar, phi, terms


def host(t):
    return t.detach().cpu().numpy()


@pytest.mark.parametrize("with_bc", [False, True])
def test_laplace_apply_and_diag(setup, with_bc):
    mesh, scalar, phi, _ = setup
    grid = Grid(BOUNDS[:2], BOUNDS[2:], (NX, NY), RULES)
    om = omodel.Heat(grid, [(1.0, [], np.ones((mesh.num_elements, 3)), None)], VOLUME)
    K = om.matrix(host(phi.values))
    bc = DirichletSet.on_tags(scalar, (2, 3)) if with_bc else None
    if with_bc:
        K, _ = ofem.dirichlet_eliminate(K, np.zeros(K.shape[0]), bc.dofs)
    op = LaplaceOperator(scalar, phi.values, 1e-3, bc)
    u = np.random.default_rng(3).standard_normal((3, K.shape[0]))
    got = host(op.apply(torch.as_tensor(u, device="cuda")))
    for g_, x in zip(got, u):
        assert rel_l2(g_, K @ x) <= 1e-12
    assert rel_l2(host(op.diagonal()), K.diagonal()) <= 1e-14


def test_states_cost_and_derivative(setup, gold):
    mesh, scalar, phi, terms = setup
    np.testing.assert_array_equal(host(phi.values), gold["phi"])
    model = HeatPlusModel(mesh, terms, VOLUME, bilinear=BIL)
    # the eliminated system carries the ground values (0) on its Dirichlet rows
    want = gold["loads"].copy()
    for t, tags in enumerate((1, (2, 3))):
        want[t, DirichletSet.on_tags(scalar, tags).dofs] = 0.0
    np.testing.assert_allclose(host(model.load_vectors), want, rtol=1e-13, atol=1e-16)
    states = lsg.solve_concurrent(model.pde(phi))
    for s, ref in zip(states, gold["states"]):
        assert rel_l2(host(s.values), ref) <= 1e-8
    # functionals on the reference's own states: 1e-10 gates
    ref_states = [FemField(scalar, torch.as_tensor(v, device="cuda")) for v in gold["states"]]
    assert model.cost(phi, ref_states) == pytest.approx(float(gold["J"][0]), rel=1e-12)
    assert model.constraint(phi, ref_states)[0] == pytest.approx(float(gold["C"][0]), rel=1e-14)
    adj = model.adjoint(phi, ref_states)
    for a, ref in zip(adj, gold["adjoints"]):
        np.testing.assert_allclose(host(a.values), ref, rtol=1e-15, atol=0)
    cost_pair, cons = model.derivative(phi, ref_states, adj)
    vc = host(cost_pair.vector[0][1])
    assert rel_l2(vc, gold["vec_cost"]) <= 1e-11
    assert rel_l2(host(cons[0].vector[0][1]), gold["vec_vol"]) <= 1e-13
    # velocity solve of the combined pair (PPL multiplier 0.41)
    vspace = FunctionSpace(mesh, 2)
    res = VelocitySolver(BIL, vspace).solve(combine_derivatives(cost_pair, cons, np.array([0.41])))
    assert rel_l2(host(res.theta.values), gold["theta"]) <= 1e-8
    assert res.form_value == pytest.approx(float(gold["form_value"][0]), rel=1e-8)


def test_single_term_without_gradient(setup, gold):
    mesh, scalar, phi, _ = setup
    model = HeatModel(mesh, 1, src_b, VOLUME, bilinear=BIL)
    (state,) = lsg.solve_concurrent(model.pde(phi))
    assert rel_l2(host(state.values), gold["single_state"]) <= 1e-8
    ref = [FemField(scalar, torch.as_tensor(gold["single_state"], device="cuda"))]
    assert model.cost(phi, ref) == pytest.approx(float(gold["single_J"][0]), rel=1e-12)
    cp, _ = model.derivative(phi, ref, model.adjoint(phi, ref))
    assert rel_l2(host(cp.vector[0][1]), gold["single_vec_cost"]) <= 1e-11


def test_terms_sharing_a_ground_are_batched(setup):
    mesh, scalar, phi, _ = setup
    terms = [HeatTerm(src_a, 1, 0.5, grad_a), HeatTerm(src_b, 1, 0.5, None)]
    model = HeatPlusModel(mesh, terms, VOLUME, bilinear=BIL)
    probs = model.pde(phi)
    assert probs[0].matrix is probs[1].matrix  # one operator -> one PCG batch
    states = lsg.solve_concurrent(probs)
    single = [lsg.solve_concurrent([p])[0] for p in probs]
    for a, b in zip(states, single):
        assert rel_l2(host(a.values), host(b.values)) <= 1e-9


def test_run_history_matches_reference_run(setup, gold):
    mesh, scalar, _, terms = setup
    phi0 = LevelSetField.from_field(scalar.interpolate(phi_fn))
    model = HeatPlusModel(mesh, terms, VOLUME, bilinear=BIL)
    params = lsg.RunParams(niter=10, start_to_check=10, reinit_step=4, reinit_pars=(8, 0.1),
                           level_set_scheme="pg")
    _, hist = lsg.run(model, phi0, params, timing=False)
    np.testing.assert_allclose([r.cost for r in hist], gold["run_cost"], rtol=1e-4)
    np.testing.assert_allclose([r.constraint[0] for r in hist], gold["run_constraint"], rtol=1e-4)
    np.testing.assert_array_equal([r.steps for r in hist], gold["run_steps"])


def test_heat_rejects_3d_and_bad_inputs():
    from paper_2601_05709_b200 import ConfigError, build_box_mesh
    box = build_box_mesh((0, 0, 0, 1, 1, 1), (2, 2, 2), [(1, lambda p: p[:, 0] < 1e-12)])
    with pytest.raises(ConfigError):
        HeatModel(box, 1, src_b, 0.5)
    mesh = build_rect_mesh(BOUNDS, 4, 4, RULES)
    with pytest.raises(ConfigError):
        HeatModel(mesh, 9, src_b, 0.5)  # no such ground tag
    with pytest.raises(ConfigError):
        HeatModel(mesh, 1, lambda p: np.full(len(p), np.nan), 0.5)
    with pytest.raises(ConfigError):
        HeatPlusModel(mesh, [HeatTerm(src_b, 1)], 0.5)

"""Inverse-elasticity model (reference ``models/inverse.py``) on the CUDA
path vs the reference's golden vectors (tests/golden/make_golden_inverse.py).

Needs a B200.  Covers the twin-data generation (fine solve, injection,
harmonic extension), the 2N batched states and adjoints, the misfit pass
(J and the adjoint right-hand sides), the S0/S1 tensors and their velocity
RHS, and a short run() history against the reference's own run().
"""

import os

import numpy as np
import pytest
import torch

from conftest import rel_l2
from inverse_cases import (BOUNDS, COARSE, CONTRAST, FINE, FIXED, FORCES, LAME, MEASURED, guess,
                           inclusion, rules)

pytestmark = pytest.mark.gpu

lsg = pytest.importorskip("paper_2601_05709_b200")
from paper_2601_05709_b200 import (BilinearSpec, ConfigError, FemField, FunctionSpace,  # noqa: E402
                                   InverseElasticityModel, LevelSetField, MeasurementPair,
                                   VelocitySolver, build_rect_mesh, dirichlet_extension,
                                   generate_measurements)
from paper_2601_05709_b200.models import resolve_adjoints  # noqa: E402


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_inverse.npz"))


@pytest.fixture(scope="module")
def meshes():
    return build_rect_mesh(BOUNDS, *COARSE, rules()), build_rect_mesh(BOUNDS, *FINE, rules())


def host(t):
    return t.detach().cpu().numpy()


def _pairs(coarse, gold):
    vec = FunctionSpace(coarse, 2)
    return [MeasurementPair(tr, tag, FemField(vec, torch.as_tensor(m, device="cuda")))
            for (tr, tag), m in zip(FORCES, gold["measured"])]


def test_twin_measurements_and_extension(meshes, gold):
    coarse, fine = meshes
    pairs = generate_measurements(fine, coarse, inclusion, FORCES, FIXED, MEASURED,
                                  contrast=CONTRAST, lame=LAME)
    for p, ref in zip(pairs, gold["measured"]):
        assert rel_l2(host(p.measured.values), ref) <= 1e-8
    vec = FunctionSpace(coarse, 2)
    tr = FemField(vec, torch.as_tensor(gold["ext_trace"], device="cuda"))
    out = dirichlet_extension(coarse, (1, 3), [tr])[0]
    assert rel_l2(host(out.values), gold["ext_out"]) <= 1e-9


def test_states_adjoints_cost_and_tensors(meshes, gold):
    coarse, _ = meshes
    scalar, vec = FunctionSpace(coarse, 1), FunctionSpace(coarse, 2)
    model = InverseElasticityModel(coarse, FIXED, MEASURED, _pairs(coarse, gold), contrast=CONTRAST,
                                   lame=LAME)
    phi = LevelSetField.from_field(scalar.interpolate(guess))
    np.testing.assert_array_equal(host(phi.values), gold["phi"])
    problems = model.pde(phi)
    assert problems[0].matrix is problems[2].matrix and problems[3].matrix is problems[5].matrix
    states = lsg.solve_concurrent(problems)
    for s, ref in zip(states, gold["states"]):
        assert rel_l2(host(s.values), ref) <= 1e-8
    # functionals on the reference's own states / adjoints: 1e-10 gates
    ref_states = [FemField(vec, torch.as_tensor(v, device="cuda")) for v in gold["states"]]
    assert model.cost(phi, ref_states) == pytest.approx(float(gold["J"][0]), rel=1e-12)
    adj_problems = model.adjoint(phi, ref_states)
    k = len(FORCES)
    want = gold["adjoint_rhs"].copy()  # eliminated systems carry 0 on their clamped rows
    want[:k, model.bc_partial.dofs] = 0.0
    want[k:, model.bc_total.dofs] = 0.0
    got = np.stack([host(p.rhs) for p in adj_problems])
    assert np.abs(got - want).max() <= 1e-12 * np.abs(want).max()
    adjoints = resolve_adjoints(model, phi, ref_states)
    for a, ref in zip(adjoints, gold["adjoints"]):
        assert rel_l2(host(a.values), ref) <= 1e-7
    ref_adj = [FemField(vec, torch.as_tensor(v, device="cuda")) for v in gold["adjoints"]]
    pair, cons = model.derivative(phi, ref_states, ref_adj)
    assert cons == []
    s0, s1 = host(pair.s0(vec)), host(pair.s1(vec))
    assert np.abs(s0 - gold["S0"]).max() <= 1e-8 * np.abs(gold["S0"]).max()
    assert np.abs(s1 - gold["S1"]).max() <= 1e-8 * np.abs(gold["S1"]).max()
    bil = BilinearSpec(mass_weight=0.1, stiffness_weight=1.0, zero_dirichlet=True)
    solver = VelocitySolver(bil, vec)
    assert rel_l2(host(solver._derivative_vector(pair)), gold["vec"]) <= 1e-8
    res = solver.solve(pair)
    assert rel_l2(host(res.theta.values), gold["theta"]) <= 1e-8


def test_run_history_matches_reference_run(meshes, gold):
    coarse, _ = meshes
    scalar = FunctionSpace(coarse, 1)
    model = InverseElasticityModel(coarse, FIXED, MEASURED, _pairs(coarse, gold), contrast=CONTRAST,
                                   lame=LAME)
    params = lsg.RunParams(niter=8, start_to_check=8, dfactor=1e-2, lv_time=(1e-3, 10.0),
                           lv_iter=(8, 32), reinit_step=5, reinit_pars=(8, 0.1), level_set_scheme="pg")
    _, hist = lsg.run(model, LevelSetField.from_field(scalar.interpolate(guess)), params, timing=False)
    np.testing.assert_allclose([r.cost for r in hist], gold["run_cost"], rtol=1e-4)
    np.testing.assert_array_equal([r.steps for r in hist], gold["run_steps"])


def test_configuration_errors(meshes, gold):
    coarse, fine = meshes
    pairs = _pairs(coarse, gold)
    with pytest.raises(ConfigError):
        InverseElasticityModel(coarse, FIXED, MEASURED, [])
    other = FemField(FunctionSpace(fine, 2), torch.zeros(2 * fine.num_vertices, dtype=torch.float64,
                                                         device="cuda"))
    with pytest.raises(ConfigError):
        InverseElasticityModel(coarse, FIXED, MEASURED, [MeasurementPair((0.0, 0.4), 3, other)])
    with pytest.raises(ConfigError):
        InverseElasticityModel(coarse, FIXED, MEASURED, pairs, alpha=-1.0)
    with pytest.raises(ConfigError):
        InverseElasticityModel(coarse, 9, MEASURED, pairs)

"""Golden vectors of the reference heat models (lsopt 0.1.0, ``models/heat.py``).

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_heat.py

Writes ``tests/golden/reference_heat.npz``: states, J, C, the S0/S1 tensors
and their contracted velocity RHS of a two-term ``HeatPlusModel`` (one
source with a spatial gradient, one constant; different grounds), a
single-term ``HeatModel``, and the history of a short reference ``run()``.
Everything comes from the reference's own public API on small inputs; only
this file travels to the GPU box.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)

from lsopt.driver import RunParams, run  # noqa: E402
from lsopt.fem import FunctionSpace  # noqa: E402
from lsopt.levelset import LevelSetField  # noqa: E402
from lsopt.mesh import build_rect_mesh  # noqa: E402
from lsopt.models import HeatModel, HeatPlusModel, HeatTerm  # noqa: E402
from lsopt.models.base import solve_problem  # noqa: E402
from lsopt.ppl import combine_derivatives  # noqa: E402
from lsopt.velocity import BilinearSpec, VelocitySolver  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_heat.npz")

BOUNDS = (0.0, 0.0, 1.5, 1.0)
NX, NY = 24, 16


def rules():
    return [(1, lambda p: p[:, 0] < 1e-12),
            (2, lambda p: (p[:, 1] < 1e-12) & (p[:, 0] > 0.5) & (p[:, 0] < 1.0)),
            (3, lambda p: p[:, 0] > 1.5 - 1e-12)]


def phi_fn(p):
    return -np.cos(4 * np.pi * p[:, 0] / 1.5) * np.cos(3 * np.pi * p[:, 1]) - 0.2


def src_a(p):
    return 1.0 + 0.5 * p[:, 0] * p[:, 1]


def grad_a(p):
    return np.stack([0.5 * p[:, 1], 0.5 * p[:, 0]], axis=1)


def src_b(p):
    return np.full(len(p), 2.0)


def terms():
    return [HeatTerm(src_a, 1, 0.7, grad_a), HeatTerm(src_b, (2, 3), None, None)]


def main():
    g = {}
    mesh = build_rect_mesh(BOUNDS, NX, NY, rules())
    scalar, vector = FunctionSpace(mesh, 1), FunctionSpace(mesh, 2)
    phi = LevelSetField.from_field(scalar.interpolate(phi_fn))
    g["phi"] = phi.values
    bil = BilinearSpec(stiffness_weight=1.0, boundary_normal_penalty=1e4)

    model = HeatPlusModel(mesh, terms(), 0.6, bilinear=bil)
    problems = model.pde(phi)
    g["loads"] = np.stack([p.rhs for p in problems])
    states = [solve_problem(p) for p in problems]
    g["states"] = np.stack([s.values for s in states])
    g["J"] = np.array([model.cost(phi, states)])
    g["C"] = np.asarray(model.constraint(phi, states))
    adj = model.adjoint(phi, states)
    g["adjoints"] = np.stack([a.values for a in adj])
    cost_pair, cons = model.derivative(phi, states, adj)
    g["S0"] = cost_pair.s0(vector)
    g["S1"] = cost_pair.s1(vector)
    solver = VelocitySolver(bil, vector)
    g["vec_cost"] = solver._derivative_vector(cost_pair)
    g["vec_vol"] = solver._derivative_vector(cons[0])
    lam = np.array([0.41])
    pair = combine_derivatives(cost_pair, cons, lam)
    res = solver.solve(pair)
    g["theta"] = res.theta.values
    g["form_value"] = np.array([res.form_value])

    single = HeatModel(mesh, 1, src_b, 0.6, bilinear=bil)
    sst = [solve_problem(p) for p in single.pde(phi)]
    g["single_state"] = sst[0].values
    g["single_J"] = np.array([single.cost(phi, sst)])
    cp1, _ = single.derivative(phi, sst, single.adjoint(phi, sst))
    g["single_vec_cost"] = solver._derivative_vector(cp1)

    # a short reference run() (driver.py:211-298) of the two-term model
    model_r = HeatPlusModel(mesh, terms(), 0.6, bilinear=bil)
    params = RunParams(niter=10, start_to_check=10, reinit_step=4, reinit_pars=(8, 0.1))
    _, hist = run(model_r, LevelSetField.from_field(scalar.interpolate(phi_fn)), params, timing=False)
    g["run_cost"] = np.array([r.cost for r in hist])
    g["run_constraint"] = np.array([float(r.constraint[0]) for r in hist])
    g["run_form_value"] = np.array([r.form_value for r in hist])
    g["run_steps"] = np.array([r.steps for r in hist])
    np.savez_compressed(OUT, **g)


if __name__ == "__main__":
    main()

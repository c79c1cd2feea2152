"""Golden vectors of the reference inverse-elasticity model (lsopt 0.1.0,
``models/inverse.py``).

Run in the build container, where the read-only reference is importable:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_inverse.py

Writes ``tests/golden/reference_inverse.npz``: twin measurements
(generate_measurements: fine solve, injection, harmonic extension), the 2N
states and 2N adjoints, J, the S0/S1 tensors and their contracted velocity
RHS, the velocity solve, and the history of a short reference ``run()``.
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
for p in (REF, os.path.dirname(HERE)):
    if p not in sys.path:
        sys.path.insert(0, p)

from inverse_cases import (BOUNDS, COARSE, CONTRAST, FINE, FIXED, FORCES, LAME, MEASURED,  # noqa: E402
                           guess, inclusion, rules)
from lsopt.driver import RunParams, run  # noqa: E402
from lsopt.fem import FunctionSpace  # noqa: E402
from lsopt.levelset import LevelSetField  # noqa: E402
from lsopt.mesh import build_rect_mesh  # noqa: E402
from lsopt.models import InverseElasticityModel  # noqa: E402
from lsopt.models.base import resolve_adjoints, solve_problem  # noqa: E402
from lsopt.models.inverse import dirichlet_extension, generate_measurements  # noqa: E402
from lsopt.velocity import BilinearSpec, VelocitySolver  # noqa: E402

OUT = os.path.join(HERE, "reference_inverse.npz")


def main():
    g = {}
    coarse = build_rect_mesh(BOUNDS, *COARSE, rules())
    fine = build_rect_mesh(BOUNDS, *FINE, rules())
    pairs = generate_measurements(fine, coarse, inclusion, FORCES, FIXED, MEASURED,
                                  contrast=CONTRAST, lame=LAME)
    g["measured"] = np.stack([p.measured.values for p in pairs])
    scalar, vector = FunctionSpace(coarse, 1), FunctionSpace(coarse, 2)
    trace = vector.interpolate(lambda p: np.stack([np.sin(p[:, 0]) + p[:, 1], p[:, 0] * p[:, 1]], 1))
    g["ext_trace"] = trace.values
    g["ext_out"] = dirichlet_extension(coarse, (1, 3), [trace])[0].values

    model = InverseElasticityModel(coarse, FIXED, MEASURED, pairs, contrast=CONTRAST, lame=LAME)
    phi = LevelSetField.from_field(scalar.interpolate(guess))
    g["phi"] = phi.values
    problems = model.pde(phi)
    g["state_rhs"] = np.stack([p.rhs for p in problems])
    states = [solve_problem(p) for p in problems]
    g["states"] = np.stack([s.values for s in states])
    g["J"] = np.array([model.cost(phi, states)])
    adj_problems = model.adjoint(phi, states)
    g["adjoint_rhs"] = np.stack([p.rhs for p in adj_problems])
    adjoints = resolve_adjoints(model, phi, states)
    g["adjoints"] = np.stack([a.values for a in adjoints])
    pair, cons = model.derivative(phi, states, adjoints)
    assert cons == []
    g["S0"] = pair.s0(vector)
    g["S1"] = pair.s1(vector)
    bil = BilinearSpec(mass_weight=0.1, stiffness_weight=1.0, zero_dirichlet=True)
    solver = VelocitySolver(bil, vector)
    g["vec"] = solver._derivative_vector(pair)
    res = solver.solve(pair)
    g["theta"] = res.theta.values
    g["form_value"] = np.array([res.form_value])

    model_r = InverseElasticityModel(coarse, FIXED, MEASURED, pairs, contrast=CONTRAST, lame=LAME)
    params = RunParams(niter=8, start_to_check=8, dfactor=1e-2, lv_time=(1e-3, 10.0), lv_iter=(8, 32),
                       reinit_step=5, reinit_pars=(8, 0.1))
    _, hist = run(model_r, LevelSetField.from_field(scalar.interpolate(guess)), params, timing=False)
    g["run_cost"] = np.array([r.cost for r in hist])
    g["run_form_value"] = np.array([r.form_value for r in hist])
    g["run_steps"] = np.array([r.steps for r in hist])
    np.savez_compressed(OUT, **g)


if __name__ == "__main__":
    main()

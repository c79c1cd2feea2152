"""The reference's own run() on the full-size BASELINE cfg1 mesh (160x80, reinit
every 5, its CN Petrov-Galerkin level-set scheme), first 30 iterations, for the
GPU run with level_set_scheme="pg".  (Run to the config's 50 iterations, the
reference's own scheme loses the design at iteration 45 -- C = 0, J = 387.6 --
and its splu fails at iteration 49 with "Factor is exactly singular"; the
north star's explicit scheme, the product default, runs all 50, see
oracle_cfg1_full.npz.)  Run in the build container (the reference is importable
there; ~1.5 min):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_cfg1_reference.py

Writes tests/golden/reference_cfg1_full.npz.
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
from lsopt.models import ComplianceModel, MaterialIndicator  # noqa: E402
from lsopt.velocity import BilinearSpec  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_cfg1_full.npz")
LAME = (0.3 / 0.91, 1.0 / 2.6)


def main():
    rules = [(1, lambda p: p[:, 0] < 1e-12),
             (2, lambda p: (p[:, 0] > 2.0 - 1e-12) & (p[:, 1] >= 0.45) & (p[:, 1] <= 0.55))]
    mesh = build_rect_mesh((0.0, 0.0, 2.0, 1.0), 160, 80, rules)
    bil = BilinearSpec(mass_weight=1.0, stiffness_weight=1e-2)
    model = ComplianceModel(mesh, 1, 2, (0.0, -1.0), 1.0, lame=LAME, bilinear=bil)
    model.material = MaterialIndicator(1.0, 1e-3)
    phi = LevelSetField.from_field(FunctionSpace(mesh, 1).interpolate(
        lambda p: -np.cos(6 * np.pi * p[:, 0]) * np.cos(4 * np.pi * p[:, 1]) - 0.4))
    params = RunParams(niter=30, start_to_check=30, reinit_step=5, reinit_pars=(8, 0.1))
    _, hist = run(model, phi, params, timing=False)
    np.savez_compressed(OUT, cost=np.array([r.cost for r in hist]),
                        constraint=np.array([float(r.constraint[0]) for r in hist]),
                        lagrangian=np.array([r.lagrangian for r in hist]),
                        form_value=np.array([r.form_value for r in hist]),
                        steps=np.array([r.steps for r in hist]),
                        t_end=np.array([r.t_end for r in hist]))
    print(len(hist), hist[0].cost, hist[-1].cost)


if __name__ == "__main__":
    main()

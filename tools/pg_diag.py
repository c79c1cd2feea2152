"""Diagnostics of the reference (PG) level-set scheme on a BASELINE config:
per outer iteration J, C, the number / iterations / residuals of the PG
solves, and max |phi| around transport and reinitialisation.

    python tools/pg_diag.py [cfg1] [niter]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05709_b200 as lsg  # noqa: E402
from paper_2601_05709_b200 import configs, driver, levelset  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
niter = int(sys.argv[2]) if len(sys.argv) > 2 else 12
c = configs.case(name)
c = type(c)(**{**c.__dict__, "niter": niter})
mesh, model, phi, params = configs.build(c)
params = lsg.RunParams(**{**params.__dict__, "level_set_scheme": "pg"})
levelset.BICG_LOG = []
notes = []
for fname in ("transport", "reinitialize"):
    orig = getattr(driver, fname)

    def wrapped(p, *a, _orig=orig, _name=fname, **k):
        out = _orig(p, *a, **k)
        notes.append((_name, float(p.values.abs().max()), float(out.values.abs().max())))
        return out

    setattr(driver, fname, wrapped)
opt = driver.Optimizer(model, phi, params, timing=False)
for it in range(niter):
    n0 = len(levelset.BICG_LOG)
    notes.clear()
    try:
        r = opt.step()
    except Exception as exc:  # report and stop
        print(it, "FAILED", type(exc).__name__, str(exc)[:200], notes, flush=True)
        break
    log = levelset.BICG_LOG[n0:]
    print(it, r.cost, float(r.constraint[0]), r.t_end, r.steps, "solves", len(log),
          "max iters", max((l[0] for l in log), default=0),
          "worst resid", max((l[1] for l in log), default=0.0), notes, flush=True)

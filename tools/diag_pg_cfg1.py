"""Print the cfg1 reference-scheme history (J, C, steps, substeps, velocity form) at full precision."""
import json, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2601_05709_b200 as lsg
from paper_2601_05709_b200 import configs
c = configs.case("cfg1")
c = type(c)(**{**c.__dict__, "niter": 10})
mesh, model, phi, params = configs.build(c)
params = lsg.RunParams(**{**params.__dict__, "level_set_scheme": "pg"})
opt = lsg.driver.Optimizer(model, phi, params, timing=False)
for _ in range(10):
    try:
        r = opt.step()
    except lsg.SolverError as e:
        print("SolverError", e); break
    print(json.dumps({"J": repr(r.cost), "C": repr(float(r.constraint[0])), "steps": r.steps,
                      "B": repr(r.form_value), "cg": [int(v) for v in r.cg_iters], "vit": r.velocity_iters,
                      "tsub": r.transport_substeps, "rsub": r.reinit_substeps}))

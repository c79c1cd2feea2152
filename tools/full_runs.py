#!/usr/bin/env python
"""Full BASELINE runs (all `niter` iterations) of cfg1, cfg2, cfg3 and cfg5 on one B200.

    python tools/full_runs.py [cfg1 cfg2 ...]

Each run builds the config (configs.py: the BASELINE text pinned as SURVEY
Appendix B says), runs the public `run()` loop for its full iteration count
and prints one JSON line: time to solution (CUDA events around the loop),
iterations/s, the first and last J and C, and the PCG iteration totals.
"""

import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2601_05709_b200 as lsg  # noqa: E402
from paper_2601_05709_b200 import configs  # noqa: E402


def main():
    names = sys.argv[1:] or ["cfg1", "cfg3", "cfg2", "cfg5"]
    for name in names:
        c = configs.case(name)
        mesh, model, phi, params = configs.build(c)
        stream = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        _, hist = lsg.run(model, phi, params, timing=False)
        e1.record(stream)
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) / 1e3
        out = {"config": name, "n": list(mesh.n), "niter": len(hist), "seconds": s,
               "iters_per_s": len(hist) / s,
               "J": [hist[0].cost, hist[-1].cost], "C": [float(hist[0].constraint[0]), float(hist[-1].constraint[0])],
               "pcg_rhs_iterations": int(sum(sum(r.cg_iters) for r in hist)),
               "velocity_iterations": int(sum(r.velocity_iters for r in hist)),
               "transport_substeps": int(sum(r.transport_substeps for r in hist))}
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()

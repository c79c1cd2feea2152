#!/usr/bin/env python
"""Per-iteration work counts of the B200 loop for the reference arm's extrapolation.

    python tools/calibrate.py [cfg1 cfg2 cfg3 cfg5] > profiles/r02_calibration.json

For each config and each bench window (W warm-up + K timed iterations; the driver's
w5k20 and bench.py's default w3k10) runs the device loop and records, averaged over
the K timed iterations: state-PCG right-hand-side iterations, H1 velocity CG
iterations, transport and reinit substeps.  bench.py --impl reference multiplies its
measured per-unit CPU costs by these counts (same algorithm and stopping rules on
both sides, so the counts agree to a few percent)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_2601_05709_b200 import configs  # noqa: E402
from paper_2601_05709_b200.driver import Optimizer  # noqa: E402

names = sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg5"]
out = {}
for name in names:
    out[name] = {}
    for W, K in ((5, 20), (3, 10)):
        c = configs.case(name)
        c = type(c)(**{**c.__dict__, "niter": W + K})
        mesh, model, phi, params = configs.build(c)
        opt = Optimizer(model, phi, params, timing=False)
        recs = [opt.step() for _ in range(W + K)][W:]
        out[name][f"w{W}k{K}"] = bench.window_counts(recs)
        print(name, W, K, out[name][f"w{W}k{K}"], file=sys.stderr, flush=True)
print(json.dumps(out, indent=1))

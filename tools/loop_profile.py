#!/usr/bin/env python
"""Where the time of one optimisation iteration goes (B200, CUDA events).

    python tools/loop_profile.py --config cfg5 [--warmup 1] [--steps 2]

Runs W + K iterations of the device-resident loop and splits the K timed
ones into state PCG (elasticity), velocity CG (H1) and the rest (material,
shape derivative, transport, reinitialisation, host PPL), with the PCG
iteration counts, using the fem.PCG_PROFILE hook.
"""

import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_05709_b200 import _lib, configs, fem  # noqa: E402
from paper_2601_05709_b200.driver import Optimizer  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--warmup", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    c = configs.case(args.config)
    c = type(c)(**{**c.__dict__, "niter": args.warmup + args.steps})
    mesh, model, phi, params = configs.build(c)
    opt = Optimizer(model, phi, params, timing=False)
    for _ in range(args.warmup):
        opt.step()
    torch.cuda.synchronize()
    fem.PCG_PROFILE = []
    lib = _lib.load()
    import ctypes
    g0 = (ctypes.c_double * 4)()
    lib.lsg_graph_stats(g0)
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs = [opt.step() for _ in range(args.steps)]
    e1.record(stream)
    torch.cuda.synchronize()
    prof, fem.PCG_PROFILE = fem.PCG_PROFILE, None
    g1 = (ctypes.c_double * 4)()
    lib.lsg_graph_stats(g1)
    total = e0.elapsed_time(e1)
    out = {"config": args.config, "steps": args.steps, "ms_per_step": total / args.steps}
    for kind, name in ((_lib.LSG_OP_ELASTICITY, "state_pcg"), (_lib.LSG_OP_H1, "velocity_cg")):
        ch = [p for p in prof if p["kind"] == kind]
        ms = sum(p["events"][0].elapsed_time(p["events"][1]) for p in ch)
        launched = sum(p["launched"] for p in ch)
        out[name] = {"ms_per_step": ms / args.steps, "launched_iters_per_step": launched / args.steps,
                     "us_per_launched_iter": 1e3 * ms / max(launched, 1),
                     "rhs_iters_per_step": sum(p["rhs_iters"] for p in ch) / args.steps,
                     "chunks_per_step": len(ch) / args.steps}
    out["graphs_per_step"] = dict(zip(("hits", "updates", "instantiations", "host_ms"),
                                      [(b - a) / args.steps * (1e3 if i == 3 else 1)
                                       for i, (a, b) in enumerate(zip(g0, g1))]))
    out["other_ms_per_step"] = out["ms_per_step"] - out["state_pcg"]["ms_per_step"] - out["velocity_cg"]["ms_per_step"]
    out["records"] = [{"cg_iters": list(r.cg_iters), "velocity_iters": r.velocity_iters,
                       "transport_substeps": r.transport_substeps, "reinit_substeps": r.reinit_substeps}
                      for r in recs]
    print(json.dumps(out))


if __name__ == "__main__":
    main()

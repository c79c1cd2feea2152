#!/usr/bin/env python
"""One optimisation iteration of a BASELINE config (+ one reinitialisation) for ncu
captures of the per-iteration kernels (shape derivative, H1 velocity CG, transport,
reinit).

    python tools/prof_loop.py [--config cfg5]
"""
import argparse
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2601_05709_b200 as lsg  # noqa: E402
from paper_2601_05709_b200 import configs  # noqa: E402
from paper_2601_05709_b200.driver import Optimizer  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="cfg5")
args = ap.parse_args()
c = configs.case(args.config)
mesh, model, phi, params = configs.build(c)
opt = Optimizer(model, phi, params, timing=False)
rec = opt.step()
lsg.reinitialize(opt.phi, 8, 0.1)
torch.cuda.synchronize()
print("ok", rec.cost, rec.transport_substeps)

#!/usr/bin/env python
"""One 3D elasticity apply (and optionally PCG iterations) for ncu captures.

    python tools/prof_apply3d.py [--grid 192x96x96] [--k 4] [--pcg 0]
"""
import argparse
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2601_05709_b200 import _lib, build_box_mesh, build_rect_mesh  # noqa: E402
from paper_2601_05709_b200.fem import DirichletSet, ElasticityOperator, FunctionSpace, _workspace  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--grid", default="192x96x96")
ap.add_argument("--k", type=int, default=4)
ap.add_argument("--pcg", type=int, default=0)
ap.add_argument("--applies", type=int, default=2)
args = ap.parse_args()
n = tuple(int(v) for v in args.grid.split("x"))
if len(n) == 3:
    mesh = build_box_mesh((0.0, 0.0, 0.0, 2.0, 1.0, 1.0), n, [(1, lambda p: p[:, 0] < 1e-12)])
    lame = (0.576923, 0.384615)
else:
    mesh = build_rect_mesh((0.0, 0.0, 2.0, 1.0), n[0], n[1], [(1, lambda p: p[:, 0] < 1e-12)])
    lame = (0.3 / 0.91, 1 / 2.6)
d, N = mesh.dim, mesh.num_vertices
space = FunctionSpace(mesh, d)
phi = torch.as_tensor(np.random.default_rng(0).standard_normal(N), device="cuda")
op = ElasticityOperator(space, phi, lame, 1e-3, DirichletSet.on_tags(space, 1))
u = torch.randn((args.k, d * N), dtype=torch.float64, device="cuda")
for _ in range(args.applies):
    op.apply(u)
if args.pcg:
    cop, st = op._op(), _lib.stream()
    ws = _workspace(op, args.k)
    ws.b.copy_(torch.randn((args.k, d * N), dtype=torch.float64, device="cuda"))
    ws.x.zero_()
    ws.ws.dinv = op.inverse_diagonal().data_ptr()
    _lib.call("lsg_pcg_start", cop, ws.ws, 0.0, 0.0, 1e12, st)
    _lib.call("lsg_pcg_iterate", cop, ws.ws, args.pcg, st)
torch.cuda.synchronize()
print("ok")

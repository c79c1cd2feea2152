#!/usr/bin/env python
"""Kernel micro-benchmarks on the B200 (CUDA events, L2 flushed where stated).

    python tools/kbench.py [--grid 1024x256] [--k 8] [--iters 200]

Times the standalone elasticity apply (k RHS), and the fused PCG iteration
(lsg_pcg_iterate with the stopping test disabled) on a random two-phase
material, and prints per-launch times and algorithmic GB/s.
"""

import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_2601_05709_b200 import _lib, build_rect_mesh, build_box_mesh  # noqa: E402
from paper_2601_05709_b200.fem import (DirichletSet, ElasticityOperator, FunctionSpace, H1Operator,  # noqa: E402
                                       _workspace)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--grid", default="1024x256")
    ap.add_argument("--k", type=int, default=8)
    ap.add_argument("--iters", type=int, default=200)
    ap.add_argument("--phi", default="random", choices=("random", "smooth"),
                    help="material: per-node random phi (every cell mixed) or cfg5's periodic holes")
    args = ap.parse_args()
    n = tuple(int(v) for v in args.grid.split("x"))
    if len(n) == 2:
        mesh = build_rect_mesh((0.0, 0.0, 4.0, 1.0), n[0], n[1], [(1, lambda p: p[:, 1] < 1e-12)])
        lame = (0.3 / 0.91, 1 / 2.6)
    else:
        mesh = build_box_mesh((0.0, 0.0, 0.0, 2.0, 1.0, 1.0), n, [(1, lambda p: p[:, 0] < 1e-12)])
        lame = (0.576923, 0.384615)
    d, N, E, k = mesh.dim, mesh.num_vertices, mesh.num_elements, args.k
    space = FunctionSpace(mesh, d)
    if args.phi == "smooth":
        v = mesh.vertices if isinstance(mesh.vertices, np.ndarray) else mesh.vertices.cpu().numpy()
        phi = torch.as_tensor(-np.prod(np.cos(6 * np.pi * v), axis=1) - 0.3, device="cuda")
    else:
        phi = torch.as_tensor(np.random.default_rng(0).standard_normal(N), device="cuda")
    op = ElasticityOperator(space, phi, lame, 1e-3, DirichletSet.on_tags(space, 1))
    stream = torch.cuda.current_stream()
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    clean = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    out = {"grid": args.grid, "k": k, "nodes": N}

    def timed(fn, reps, flush_l2):
        # The whole sequence is queued behind a ~50 ms device sleep so that
        # the GPU never waits on the host between e0 and the kernel: the
        # events bracket device time only (not the Python/ctypes launch).
        torch.cuda.synchronize()
        torch.cuda._sleep(100_000_000)
        evs = []
        for rep in range(reps + 3):
            if flush_l2:
                flush.fill_(float(rep))
                if flush_l2 == "clean":  # write back the flush's dirty lines before the launch
                    clean.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            fn()
            e1.record(stream)
            if rep >= 3:
                evs.append((e0, e1))
        torch.cuda.synchronize()
        return float(np.median([a.elapsed_time(b) * 1e3 for a, b in evs]))

    u = torch.randn((k, d * N), dtype=torch.float64, device="cuda")
    y = torch.empty_like(u)
    cop = op._op()
    st = _lib.stream()
    apply = lambda: _lib.call("lsg_apply", cop, k, _lib.ptr(u), _lib.ptr(y), st)
    for name, fl in (("apply_cold_us", True), ("apply_clean_us", "clean"), ("apply_warm_us", False)):
        t = timed(apply, 20, fl)
        out[name] = t
        out[name.replace("_us", "_frac")] = (16.0 * d * k * N + E) / (t * 1e-6) / 1e9 / peak
    # fused PCG iterations, stopping disabled (rtol = atol = 0)
    ws = _workspace(op, k)
    ws.b.copy_(torch.randn((k, d * N), dtype=torch.float64, device="cuda"))
    ws.x.zero_()
    ws.ws.dinv = op.inverse_diagonal().data_ptr()
    _lib.call("lsg_pcg_start", cop, ws.ws, 0.0, 0.0, 1e12, st)
    it = args.iters
    t = timed(lambda: _lib.call("lsg_pcg_iterate", cop, ws.ws, it, st), 3, False) / it
    bytes_it = (80.0 * k + 16.0) * d * N + E
    out["pcg_iter_us"] = t
    out["pcg_gbs"] = bytes_it / (t * 1e-6) / 1e9
    out["pcg_frac"] = out["pcg_gbs"] / peak
    # the velocity form's PCG iteration (mass + alpha vector Laplacian, one right-hand side)
    h1 = H1Operator(space, 1.0, 1e-2)
    hws = _workspace(h1, 1)
    hws.b.copy_(torch.randn((1, d * N), dtype=torch.float64, device="cuda"))
    hws.x.zero_()
    hws.ws.dinv = h1.inverse_diagonal().data_ptr()
    hop = h1._op()
    _lib.call("lsg_pcg_start", hop, hws.ws, 0.0, 0.0, 1e12, st)
    out["h1_pcg_iter_us"] = timed(lambda: _lib.call("lsg_pcg_iterate", hop, hws.ws, it, st), 3, False) / it
    print(json.dumps(out))


if __name__ == "__main__":
    main()

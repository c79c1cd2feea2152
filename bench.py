#!/usr/bin/env python
"""Benchmark of the level-set compliance loop on B200 (see DESIGN.md section "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config cfg2]

One step = one optimisation iteration of the full loop (batched state PCG,
compliance + shape derivative, H1 velocity solve, transport, reinit every 5)
on BASELINE.json configs[1] (cfg2: 1024x256 bridge, 8 load cases).  Prints
one JSON line on rank 0.  N > 1 runs N independent replicas (one per GPU,
"replicas only": the north star is single-GPU; no collective on the data path).
"""

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "optimization iters/sec"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0
# Mean state-PCG right-hand-side iterations per outer iteration of cfg2 over
# the default window (iterations 3..12), measured by this bench on B200
# (profiles/r01_bench_notes.md); used to extrapolate the bounded CPU sample to
# a whole iteration.  Same algorithm and stopping rule on both sides.
CFG2_RHS_ITERS_PER_OUTER = 127687.0
# PCG right-hand-side iterations per outer iteration measured on the B200 runs
# (tools/loop_profile.py; cfg4 = its one solve to 1e-8), used to extrapolate the
# bounded CPU samples of the reference arm
RHS_ITERS_PER_OUTER = {"cfg1": 2132.0, "cfg2": CFG2_RHS_ITERS_PER_OUTER, "cfg3": 2200.0,
                       "cfg4": 197320.0, "cfg5": 17079.0}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-largest", action="store_true",
                    help="skip the apply measurements on the largest 2D / 3D meshes (cfg4, cfg5)")
    ap.add_argument("--shard-loads", action="store_true",
                    help="N > 1: split the load cases across GPUs (strong scaling, one NCCL "
                         "all-reduce of J and the derivative vector per iteration) instead of "
                         "running independent replicas")
    return ap.parse_args()


def largest_applies(hbm, fp64_peak):
    """The north star's apply gate on the largest meshes: cfg4 (2D, 4096x2048, k = 1) and
    cfg5 (3D, 192x96x96 Kuhn tets, k = 4), random two-phase material, clamped x = 0,
    L2 flushed (256 MB write + read) before each launch.  Bytes: 16 d k N + material."""
    import torch

    from paper_2601_05709_b200 import build_box_mesh, build_rect_mesh
    from paper_2601_05709_b200.fem import DirichletSet, ElasticityOperator, FunctionSpace

    out = {}
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    clean = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    for name, dim, n, k in (("cfg4", 2, (4096, 2048), 1), ("cfg5", 3, (192, 96, 96), 4)):
        rule = [(1, lambda p: p[:, 0] < 1e-12)]
        if dim == 2:
            mesh = build_rect_mesh((0.0, 0.0, 2.0, 1.0), n[0], n[1], rule)
            lame = (0.3 / 0.91, 1.0 / 2.6)
        else:
            mesh = build_box_mesh((0.0, 0.0, 0.0, 2.0, 1.0, 1.0), n, rule)
            lame = (0.3 / (1.3 * 0.4), 1.0 / 2.6)
        N, E = mesh.num_vertices, mesh.num_elements
        space = FunctionSpace(mesh, dim)
        phi = torch.as_tensor(np.random.default_rng(0).standard_normal(N), device="cuda")
        op = ElasticityOperator(space, phi, lame, 1e-3, DirichletSet.on_tags(space, 1))
        u = torch.randn((k, dim * N), dtype=torch.float64, device="cuda")
        op.apply(u)
        torch.cuda.synchronize()
        torch.cuda._sleep(100_000_000)
        evs = []
        for rep in range(13):
            flush.fill_(float(rep))
            clean.sum()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            op.apply(u)
            a1.record(stream)
            if rep >= 3:
                evs.append((a0, a1))
        torch.cuda.synchronize()
        t = statistics.median([e0.elapsed_time(e1) / 1e3 for e0, e1 in evs])
        byts = 16.0 * dim * k * N + (E if dim == 2 else 4.0 * N)
        out[name] = {"grid": "x".join(map(str, n)), "k": k, "ms": t * 1e3,
                     "dof_per_s": k * dim * N / t, "gbs": byts / t / 1e9,
                     "frac": byts / t / 1e9 / hbm, "bytes": byts}
        del op, u
    # Kuhn-tet stencil: ~220 fp64 instructions per cell and field
    cells = 192 * 96 * 96
    lanes = 220.0 * cells * 4
    t_fp64 = lanes / ((fp64_peak or 34.172e12) / 2)  # DFMA lane-ops/s = FLOP/s / 2
    out["cfg5"]["fp64_bound_ms"] = t_fp64 * 1e3
    out["cfg5"]["fp64_pipe_frac"] = t_fp64 / (out["cfg5"]["ms"] / 1e3)
    out["cfg5"]["note"] = ("fp64-issue-bound: ~220 fp64 instructions per cell and field need %.0f us "
                           "at the measured fp64 peak, which caps the HBM fraction near 0.6 even at "
                           "100%% of the fp64 pipe; fp64_pipe_frac is this op count over the "
                           "measured time" % (t_fp64 * 1e6))
    del flush, clean
    return out


def ncu_traffic():
    """DRAM bytes per fused PCG iteration from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_ncu_pcg_rq.json")) as f:
            return float(json.load(f)["traffic_bytes_per_pcg_iteration"])
    except Exception:
        return None


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def dist_info():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


# ---------------------------------------------------------------------------------------------
# CPU baseline: the oracle (numpy/scipy restatement of the reference path) on a bounded sample
# ---------------------------------------------------------------------------------------------

def cpu_sample(c, cg_iters_per_load, threads):
    """Time one bounded outer iteration of the oracle on config c.

    Measured: assembly + Dirichlet elimination of the shared operator (all
    loads), ``cg_iters_per_load`` Jacobi-PCG iterations per load (scipy cg, as
    the reference, fem.py:306; loads on ``threads`` threads like the
    reference's task_parallel mode, driver.py:185), the S1 tensor + derivative
    vector, and one transport call of the explicit scheme.  Not measured (so
    the CPU figure is optimistic): the velocity form's one-time SuperLU
    factorisation and per-iteration triangular solves, and reinitialisation.
    Returns dict of seconds.
    """
    from concurrent.futures import ThreadPoolExecutor

    from oracle import cases as ocases, fem as ofem, levelset as olevel, model as omodel

    grid, model, _, phi, _, h = ocases.build(c, velocity=False)
    t0 = time.perf_counter()
    systems = model.eliminated(phi)
    t_asm = time.perf_counter() - t0

    def one(args):
        A, b = args
        try:
            ofem.jacobi_pcg(A, b, maxiter=cg_iters_per_load)
        except ofem.SolverError:
            pass

    t0 = time.perf_counter()
    if threads > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(one, systems))
    else:
        for s in systems:
            one(s)
    t_cg = time.perf_counter() - t0
    states = [np.sin(np.arange(model.space.dof_count) * (1e-3 * (k + 1))) * 1e-3
              for k in range(len(systems))]
    t0 = time.perf_counter()
    s1 = model.s1_combined(phi, states, 0.5)
    vec = omodel.derivative_vector(model.space, s1=s1)
    t_s1 = time.perf_counter() - t0
    theta = -vec / (np.abs(vec).max() + 1e-30)
    t0 = time.perf_counter()
    _, nsub = olevel.transport(grid, phi, theta, 1e-3, 8, False, h)
    t_tr = time.perf_counter() - t0
    # the reference's apply: its assembled, eliminated CSR operator times the k fields
    A = systems[0][0]
    U = np.random.default_rng(0).standard_normal((A.shape[0], len(systems)))
    A @ U
    t0 = time.perf_counter()
    for _ in range(5):
        A @ U
    t_apply = (time.perf_counter() - t0) / 5
    return {"asm": t_asm, "cg": t_cg, "cg_rhs_iters": cg_iters_per_load * len(systems),
            "s1": t_s1, "transport": t_tr, "k": len(systems), "n": model.space.dof_count,
            "apply": t_apply}


def cpu_iters_per_sec(s, rhs_iters_per_outer):
    per_rhs_iter = s["cg"] / s["cg_rhs_iters"]
    t_outer = s["asm"] + per_rhs_iter * rhs_iters_per_outer + s["s1"] + s["transport"]
    return 1.0 / t_outer, t_outer


# ---------------------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------------------

def b200_arm(args, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2601_05709_b200 as lsg
    from paper_2601_05709_b200 import _lib, configs, fem
    from paper_2601_05709_b200.driver import Optimizer

    torch.cuda.set_device(local)
    lib = _lib.load()
    c = configs.case(args.config)
    W, K = args.warmup, args.steps
    c = type(c)(**{**c.__dict__, "niter": W + K})
    mesh, model, phi, params = configs.build(c)
    sharded = bool(args.shard_loads and world > 1)
    if sharded:
        from paper_2601_05709_b200.parallel import ShardedCompliance
        model = ShardedCompliance(model)
    d, N, E = mesh.dim, mesh.num_vertices, mesh.num_elements
    k = int(model.load_vectors.shape[0])

    def barrier():
        if world > 1:
            dist.barrier()

    # ---- device-resident loop: W warm-up + K timed optimisation iterations ----------------
    opt = Optimizer(model, phi, params, timing=False)
    for _ in range(W):
        opt.step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    fem.PCG_PROFILE = []
    launches0 = lib.lsg_launch_count()
    clocks = ClockSampler(local)
    clocks.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs = [opt.step() for _ in range(K)]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    clk = clocks.stop()
    launches = lib.lsg_launch_count() - launches0
    prof, fem.PCG_PROFILE = fem.PCG_PROFILE, None
    t_local = e0.elapsed_time(e1) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    value = (1 if sharded else world) * K / t_max

    # ---- roofline of the dominant kernel pair: the fused PCG iteration ----------------
    # (80 k + 16) d N + E bytes per iteration of k right-hand sides.
    state_chunks = [p for p in prof if p["kind"] == _lib.LSG_OP_ELASTICITY]
    pcg_ms = sum(p["events"][0].elapsed_time(p["events"][1]) for p in state_chunks)
    rhs_iters = sum(p["rhs_iters"] for p in state_chunks)
    launched_iters = sum(p["launched"] for p in state_chunks)
    max_iters = sum(p["max_iters"] for p in state_chunks)
    pcg_bytes = 80.0 * d * N * rhs_iters + (16.0 * d * N + E) * max_iters
    hbm, peak_kind = peaks()
    achieved = pcg_bytes / (pcg_ms / 1e3) / 1e9 if pcg_ms > 0 else 0.0
    all_ms = sum(p["events"][0].elapsed_time(p["events"][1]) for p in prof)

    # ---- standalone elasticity apply (k = 8), L2 flushed between launches ------------------
    # Flush = a 256 MB write (evicts every line the apply touched), then a 256 MB read of
    # another buffer so that the flush's dirty lines are written back before the timed
    # launch instead of inside it.  Both runs are reported; `ms` is the clean-flush one.
    op = opt.model.operator(opt.phi)
    u = torch.randn((k, d * N), dtype=torch.float64, device="cuda")
    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    clean = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")

    def apply_times(clean_flush):
        # queued behind a device sleep: the events bracket device time, not the host launch
        torch.cuda.synchronize()
        torch.cuda._sleep(100_000_000)
        evs = []
        for rep in range(23):
            flush.fill_(float(rep))
            if clean_flush:
                clean.sum()
            a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a0.record(stream)
            op.apply(u)
            a1.record(stream)
            if rep >= 3:
                evs.append((a0, a1))
        torch.cuda.synchronize()
        return statistics.median([e0.elapsed_time(e1) / 1e3 for e0, e1 in evs])

    t_apply_dirty = apply_times(False)
    t_apply = apply_times(True)
    del flush, clean
    apply_bytes = 16.0 * d * k * N + E

    largest = None
    if not args.no_largest and rank == 0:
        fp64 = None
        try:
            with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as f:
                fp64 = float(json.load(f)["fp64_tflops"]) * 1e12
        except Exception:
            fp64 = None
        largest = largest_applies(hbm, fp64)

    # ---- end to end through the public API from host buffers ----------------------------
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        barrier()
        phi_host = torch.from_numpy(np.ascontiguousarray(c.phi0(mesh.vertices), dtype=np.float64)).pin_memory()
        loads_host = model.load_vectors.cpu().pin_memory()
        out_host = torch.empty(N, dtype=torch.float64).pin_memory()
        d2h = [0]

        def on_record(rec, phi_dev):
            out_host.copy_(phi_dev.values, non_blocking=False)
            d2h[0] += N * 8 + 8 * 8

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m2, model2, _, params2 = configs.build(c)          # loads assembled host-side, uploaded
        model2._loads.copy_(loads_host, non_blocking=True)  # explicit pinned H2D of the loads
        phi_dev = lsg.LevelSetField.from_field(
            lsg.FemField(lsg.FunctionSpace(m2, 1), phi_host.to("cuda", non_blocking=True)))
        lsg.run(model2, phi_dev, params2, on_record=on_record, timing=False)
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        te = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        n_it = W + K
        h2d = (phi_host.numel() + loads_host.numel()) * 8
        e2e = {"value": world * n_it / float(te.item()), "unit": "iters/s",
               "h2d_bytes_per_step": int(h2d / n_it), "d2h_bytes_per_step": int(d2h[0] / n_it),
               "iterations": n_it,
               "note": "public run() from pinned host phi0/loads, niter=W+K incl. the cold-start "
                       "first iterations; phi + record read back to host every iteration"}

    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------------
    cpu = None
    rhs_per_outer = sum(sum(r.cg_iters) for r in recs) / K
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        s = cpu_sample(c, cg_iters_per_load=25, threads=1)
        v, t_outer = cpu_iters_per_sec(s, rhs_per_outer)
        cpu = {"value": v, "unit": "iters/s", "cores": 1, "kind": "port",
               "apply_dof_per_s": s["k"] * s["n"] / s["apply"],
               "breakdown": {"assembly_s": s["asm"], "pcg_ms_per_rhs_iteration": s["cg"] / s["cg_rhs_iters"] * 1e3,
                             "s1_and_rhs_s": s["s1"], "transport_s": s["transport"]},
               "apply_note": "scipy CSR (the reference's assembled, Dirichlet-eliminated operator) "
                             "times the k load-case fields, 1 thread; assembly not included",
               "sample": f"oracle (numpy/scipy restatement of the reference path) on {args.config}: "
                         f"assembly+elimination, 25 scipy-cg Jacobi-PCG iterations x {s['k']} loads, "
                         f"S1 + derivative vector, one transport; extrapolated to "
                         f"{rhs_per_outer:.0f} PCG rhs-iterations/outer iteration measured here; "
                         f"velocity LU + reinit not counted (CPU figure optimistic); "
                         f"{s['cg'] / s['cg_rhs_iters'] * 1e3:.2f} ms per PCG rhs-iteration, "
                         f"{t_outer:.1f} s per outer iteration"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": 1e3 * t_max / K, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{args.config}: 2D bridge 1024x256 P1 (526,850 dofs), 8 load "
                                   "cases batched, full loop (state PCG rtol 1e-10, S1+RHS, H1 CG, "
                                   "transport, reinit every 5)",
                       "nodes": N, "elements": E, "load_cases": k,
                       "l2": "PCG working set (x,r,p,q for 8 rhs = 135 MB) exceeds the 126 MB L2; "
                             "standalone apply timings flush L2 with a 256 MB write (+ a 256 MB "
                             "read that cleans it) before each launch",
                       "parallelism": (f"load cases sharded over {world} GPUs" if sharded else
                                       f"replicas x{world}" if world > 1 else "single GPU")},
            "roofline": {"bound": "hbm", "kernel": "single-pass PCG iteration march_pcg_rqs "
                                                   "(r, z, p, x of iteration i and q_i = A p_i in one "
                                                   "launch; q_{i-1} = A p_{i-1} recomputed, not stored)",
                         "achieved": achieved, "peak": hbm, "unit": "GB/s",
                         "frac": achieved / hbm, "traffic": ncu_traffic(),
                         "traffic_note": "DRAM bytes of one PCG iteration (one launch) from "
                                         "profiles/r01_ncu_pcg_rq.json (cold cache): below the "
                                         "algorithmic (canonical two-pass, 10 vectors per rhs) "
                                         "count because the pass moves 6 vectors per rhs (q is "
                                         "recomputed, x updated in the same pass) and some writes "
                                         "stay in L2; achieved/peak is the canonical-byte rate, the "
                                         "actual DRAM rate is traffic / launch time",
                         "peak_kind": peak_kind,
                         "bytes_per_iteration": "(80k+16) d N + E per k-rhs iteration",
                         "pcg_ms_in_timed_region": pcg_ms, "pcg_share_of_step": all_ms / (t_local * 1e3),
                         "rhs_iterations": rhs_iters, "launched_iterations": launched_iters},
            "apply": {"k": k, "ms": t_apply * 1e3, "dof_per_s": k * d * N / t_apply,
                      "gbs": apply_bytes / t_apply / 1e9, "frac": apply_bytes / t_apply / 1e9 / hbm,
                      "bytes": apply_bytes, "ms_dirty_flush": t_apply_dirty * 1e3,
                      "flush": "256 MB write + 256 MB read of another buffer before each launch "
                               "(ms_dirty_flush: write only; the flush's dirty lines are then "
                               "written back during the timed launch)"},
            "apply_largest": largest,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clk,
            "history": {"J": [r.cost for r in recs], "C": [float(r.constraint[0]) for r in recs],
                        "rhs_pcg_iters_per_outer": rhs_per_outer,
                        "velocity_iters": [r.velocity_iters for r in recs]},
        }
        print(json.dumps(line), flush=True)


def reference_arm(args, world, rank, local):
    """The reference path on the host: the oracle port (numpy/scipy restatement of
    lsopt's algorithm; the reference is Python and does not travel to the GPU box).
    Each step is a bounded sample of one cfg2 outer iteration, extrapolated."""
    if rank != 0:
        return
    from paper_2601_05709_b200 import configs

    c = configs.case(args.config)
    threads = min(8, os.cpu_count() or 1)
    vals = []
    for i in range(args.warmup + args.steps):
        s = cpu_sample(c, cg_iters_per_load=10, threads=threads)
        v, t_outer = cpu_iters_per_sec(s, RHS_ITERS_PER_OUTER[args.config])
        if i >= args.warmup:
            vals.append(t_outer)
    t_outer = statistics.median(vals)
    v = 1.0 / t_outer
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_outer * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{args.config} (same as the b200 arm)"},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": "per step: oracle assembly + 10 scipy-cg PCG iterations per load "
                                   f"({threads} threads, reference task_parallel mode) + S1/RHS + "
                                   f"transport, extrapolated with {RHS_ITERS_PER_OUTER[args.config]:.0f} "
                                   "PCG rhs-iterations per outer iteration"},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local = dist_info()
    if args.impl == "reference":
        reference_arm(args, world, rank, local)
        return
    if world > 1:
        import torch
        import torch.distributed as dist

        torch.cuda.set_device(local)
        dist.init_process_group("nccl")
    b200_arm(args, world, rank, local)
    if world > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()

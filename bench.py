#!/usr/bin/env python
"""Benchmark of the level-set compliance loop on B200 (see DESIGN.md section "Measurement").

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference] [--config cfg5]

One step = one optimisation iteration of the full loop (batched state PCG,
compliance + shape derivative, H1 velocity solve, transport, reinit every 5).
The default workload is BASELINE.json configs[4] (cfg5: 192x96x96 Kuhn box,
5.4M dofs, 4 load cases batched) -- the largest full-loop configuration on one
GPU; cfg2 (the 2D bridge, configs[1]) is reported beside it as `secondary`.
Prints one JSON line on rank 0.  N > 1 runs N independent replicas (one per
GPU, "replicas only": the north star is single-GPU; no collective on the data
path).

`--impl reference` times the reference's CPU algorithm (the numpy/scipy oracle:
the reference itself is Python and does not travel to the GPU box) on bounded
samples of the same workload and extrapolates to whole iterations with the
per-iteration counts the B200 arm measured in the same window
(profiles/r02_calibration.json); the extrapolation is an explicit field and
`ms_per_step` is the time each step really took.
"""

import os

# one BLAS thread per process for the CPU legs: the oracle's scipy cg is a chain of
# small BLAS calls, which threaded OpenBLAS slows down ~50x on a shared host
for _v in ("OPENBLAS_NUM_THREADS", "OMP_NUM_THREADS", "MKL_NUM_THREADS"):
    os.environ.setdefault(_v, "1")

import argparse  # noqa: E402
import json  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import tempfile  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "optimization iters/sec"
PEAKS_FILE = os.path.join(ROOT, "MEASURED_PEAKS.json")
CALIBRATION = os.path.join(ROOT, "profiles", "r02_calibration.json")
NCU_SUMMARY = os.path.join(ROOT, "profiles", "r02_ncu_kernels.json")
FALLBACK_HBM = 6650.0

WORKLOAD = {
    "cfg1": "cfg1: 2D cantilever 160x80 P1 (26,082 dofs), 1 load case",
    "cfg2": "cfg2: 2D bridge 1024x256 P1 (526,850 dofs), 8 load cases batched",
    "cfg3": "cfg3: 3D cantilever 96x48x48 Kuhn tets (698,691 dofs), 1 load case",
    "cfg4": "cfg4: 2D stress test 4096x2048 P1 (16.8M dofs), body force, 1 load case",
    "cfg5": "cfg5: 3D box 192x96x96 Kuhn tets (5,447,811 dofs), 4 load cases batched",
}
PCG_KERNELS = {2: "single-pass 2D PCG iteration march_pcg_rqs (r, z, p, x of iteration i and "
                  "q_i = A p_i in one launch; q_{i-1} recomputed, not stored)",
               3: "3D PCG iteration = pcg_prep (p = M^-1 r + beta p, pending x updates) + "
                  "march3s<ElastC,PCGQ> (q = A p, p.q) + pcg_update (r -= alpha q, r.M^-1 r, r.r); "
                  "a batch runs as two halves on two streams"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-secondary", action="store_true", help="skip the cfg2 loop beside the headline")
    ap.add_argument("--no-largest", action="store_true",
                    help="skip the apply measurements on the largest 2D / 3D meshes (cfg4, cfg5)")
    ap.add_argument("--shard-loads", action="store_true",
                    help="N > 1: split the load cases across GPUs (strong scaling, one NCCL "
                         "all-reduce of J and the derivative vector per iteration) instead of "
                         "running independent replicas")
    return ap.parse_args()


def peaks():
    try:
        with open(PEAKS_FILE) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return FALLBACK_HBM, "fallback"


def ncu_kernels():
    """Committed ncu --set full counters per kernel (profiles/r02_ncu_kernels.json)."""
    try:
        with open(NCU_SUMMARY) as f:
            return json.load(f)
    except Exception:
        return {}


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
# CPU side: the oracle (numpy/scipy restatement of the reference path) on bounded samples
# ---------------------------------------------------------------------------------------------

_SYS = None


def _cg_sample(args):
    """Seconds per scipy-cg iteration, setup excluded (difference of two runs of n and
    2n iterations, n grown until the longer run takes >= 0.2 s)."""
    from oracle import fem as ofem
    A, b, iters = _SYS

    def run(n):
        t0 = time.perf_counter()
        try:
            ofem.jacobi_pcg(A, b, rtol=0.0, atol=0.0, maxiter=n)
        except ofem.SolverError:
            pass
        return time.perf_counter() - t0

    n = iters
    while True:
        t1, t2 = run(n), run(2 * n)
        if t2 >= 0.2 or n >= 4096:
            return max(t2 - t1, 1e-9) / n
        n *= 4


def cpu_units(c, procs, slab=None, cg_iters=6, vel_iters=6):
    """Per-unit costs of one outer iteration of the reference's CPU algorithm on config c.

    Measured on a slab of the config's own mesh (same cell size; full x-y
    extent, `slab` cells along the last axis) and scaled by the element ratio:
    every oracle operation here is a sweep over elements or CSR rows, linear in
    the mesh size.  Units: assembly + Dirichlet elimination of the shared
    operator for all loads (reference fem.py:141-150,274-291, once per
    iteration), one scipy-cg Jacobi-PCG iteration per right-hand side
    (fem.py:294-316; `procs` right-hand sides run concurrently in forked
    processes, the most the reference's task-parallel mode could use), S1 +
    derivative vector (compliance.py:128-139, velocity.py:129-142), one CG
    iteration of the H1 velocity form (3D; velocity.py:98-154 factors it with
    SuperLU, out of reach at 3D sizes), one transport substep and one reinit
    substep of the explicit scheme (the north star's level-set update)."""
    import multiprocessing as mp

    from oracle import cases as ocases, levelset as olevel, model as omodel

    global _SYS
    n = tuple(c.n)
    full_cells = float(np.prod(n))
    if slab is None:
        slab = max(1, int(round(n[-1] / 48))) if c.dim == 3 else max(2, int(round(n[-1] / 16)))
    slab = min(slab, n[-1])
    h_last = (c.hi[-1] - c.lo[-1]) / n[-1]
    # slab of the mesh; clamp on x = lo and the k load cases on the x = hi face, so that
    # every slab has both (the timed costs do not depend on where the patches sit)
    x0, x1 = c.lo[0], c.hi[0]
    patch = (lambda p: p[:, 0] > x1 - 1e-12)
    sc = type(c)(**{**c.__dict__, "n": n[:-1] + (slab,),
                    "hi": tuple(c.hi[:-1]) + (c.lo[-1] + slab * h_last,),
                    "fixed": (lambda p: p[:, 0] < x0 + 1e-12),
                    "loads": tuple((g, patch) for g, _ in c.loads)})
    scale = full_cells / float(np.prod(sc.n))
    grid, model, _, phi, _, h = ocases.build(sc, velocity=False)
    rng = np.random.default_rng(0)
    out = {"slab": "x".join(map(str, sc.n)), "scale": scale}
    t0 = time.perf_counter()
    systems = model.eliminated(phi)
    out["assembly_s"] = (time.perf_counter() - t0) * scale
    A = systems[0][0]
    p = max(1, min(procs, len(systems)))
    _SYS = (A, rng.standard_normal(A.shape[0]), cg_iters)
    if p > 1:  # concurrent right-hand sides; each worker times its own iterations
        with mp.get_context("fork").Pool(p) as pool:
            wall = max(pool.map(_cg_sample, range(p)))
    else:
        wall = _cg_sample(0)
    _SYS = None
    out["pcg_rhs_iter_s"] = wall / p * scale
    out["pcg_procs"] = p
    states = [rng.standard_normal(model.space.dof_count) * 1e-3 for _ in systems]
    t0 = time.perf_counter()
    s1 = model.s1_combined(phi, states, 0.5)
    vec = omodel.derivative_vector(model.space, s1=s1)
    out["s1_rhs_s"] = (time.perf_counter() - t0) * scale
    vel = omodel.Velocity(grid, mass_weight=c.h1[0], stiffness_weight=c.h1[1], direct=False)
    B = vel.solvable
    m = vel_iters
    while True:
        tv = []
        for mm in (m, 2 * m):
            t0 = time.perf_counter()
            omodel._jacobi_cg(B, -vec, 0.0, maxiter=mm)
            tv.append(time.perf_counter() - t0)
        if tv[1] >= 0.2 or m >= 4096:
            break
        m *= 4
    vel_iters = m
    out["velocity_iter_s"] = max(tv[1] - tv[0], 1e-9) / vel_iters * scale
    theta = -vec / (np.abs(vec).max() + 1e-30)
    t0 = time.perf_counter()
    _, nsub = olevel.transport(grid, phi, theta, 1e-9, 2, False, h)
    out["transport_substep_s"] = (time.perf_counter() - t0) / nsub * scale
    t0 = time.perf_counter()
    _, nr = olevel.reinitialize(grid, phi, 2, 1e-9, h)
    out["reinit_substep_s"] = (time.perf_counter() - t0) / nr * scale
    return out


def cpu_seconds_per_iteration(u, counts):
    """Extrapolate the per-unit costs to one outer iteration with measured counts."""
    return (u["assembly_s"] + u["pcg_rhs_iter_s"] * counts["rhs_pcg_iters"] + u["s1_rhs_s"]
            + u["velocity_iter_s"] * counts["velocity_iters"]
            + u["transport_substep_s"] * counts["transport_substeps"]
            + u["reinit_substep_s"] * counts["reinit_substeps"])


def window_counts(recs):
    n = max(len(recs), 1)
    return {"rhs_pcg_iters": sum(sum(r.cg_iters) for r in recs) / n,
            "velocity_iters": sum(r.velocity_iters for r in recs) / n,
            "transport_substeps": sum(r.transport_substeps for r in recs) / n,
            "reinit_substeps": sum(r.reinit_substeps for r in recs) / n}


# ---------------------------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------------------------

def flushed_apply_ms(op, u, reps=13):
    """Median standalone apply time, L2 flushed (256 MB write + 256 MB read of another
    buffer, so the flush's dirty lines are written back before the timed launch)."""
    import torch

    flush = torch.empty(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    clean = torch.ones(256 * 1024 * 1024 // 8, dtype=torch.float64, device="cuda")
    stream = torch.cuda.current_stream()
    op.apply(u)
    torch.cuda.synchronize()
    torch.cuda._sleep(100_000_000)  # events bracket device time, not host launches
    evs = []
    for rep in range(reps):
        flush.fill_(float(rep))
        clean.sum()
        a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a0.record(stream)
        op.apply(u)
        a1.record(stream)
        if rep >= 3:
            evs.append((a0, a1))
    torch.cuda.synchronize()
    del flush, clean
    return statistics.median([e0.elapsed_time(e1) for e0, e1 in evs])


def largest_applies(hbm, ncu):
    """The north star's apply gate on the largest meshes: cfg4 (2D, 4096x2048, k = 1) and
    cfg5 (3D, 192x96x96 Kuhn tets, k = 4), random two-phase material, clamped x = 0.
    Bytes: 16 d k N + E (material 1 B per element)."""
    import torch

    from paper_2601_05709_b200 import _lib, build_box_mesh, build_rect_mesh
    from paper_2601_05709_b200.fem import DirichletSet, ElasticityOperator, FunctionSpace, _workspace

    out = {}
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
        ms = flushed_apply_ms(op, u)
        byts = 16.0 * dim * k * N + E
        kern = {key: v for key, v in ncu.get(f"apply_{name}", {}).items() if key != "launches"}
        out[name] = {"grid": "x".join(map(str, n)), "k": k, "ms": ms, "dof_per_s": k * dim * N / (ms / 1e3),
                     "gbs": byts / (ms / 1e3) / 1e9, "frac": byts / (ms / 1e3) / 1e9 / hbm, "bytes": byts,
                     "ncu": kern or None}
        # the fused PCG iteration standalone (stopping disabled: rtol = atol = 0), the north
        # star's "fused CG >= 60% of HBM on the largest meshes"; (80k+16) d N + E bytes
        ws = _workspace(op, k)
        ws.b.copy_(torch.randn((k, dim * N), dtype=torch.float64, device="cuda"))
        ws.x.zero_()
        ws.ws.dinv = op.inverse_diagonal().data_ptr()
        cop, st = op._op(), _lib.stream()
        _lib.call("lsg_pcg_start", cop, ws.ws, 0.0, 0.0, 1e12, st)
        _lib.call("lsg_pcg_iterate", cop, ws.ws, 32, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        _lib.call("lsg_pcg_iterate", cop, ws.ws, 64, st)
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 64
        pbytes = (80.0 * k + 16.0) * dim * N + E
        out[name]["pcg"] = {"us_per_iteration": us, "gbs": pbytes / (us * 1e-6) / 1e9,
                            "frac": pbytes / (us * 1e-6) / 1e9 / hbm, "bytes": pbytes,
                            "note": "standalone fused PCG iteration (64 iterations after 32, stopping "
                                    "disabled), canonical two-pass bytes"}
        del op, u, ws
    return out


def loop_window(c, W, K, world, sharded, dist):
    """W untimed + K device-timed optimisation iterations; returns the timing record."""
    import torch

    from paper_2601_05709_b200 import _lib, configs, fem
    from paper_2601_05709_b200.driver import Optimizer

    lib = _lib.load()
    c = type(c)(**{**c.__dict__, "niter": W + K})
    mesh, model, phi, params = configs.build(c)
    if sharded:
        from paper_2601_05709_b200.parallel import ShardedCompliance
        model = ShardedCompliance(model)
    opt = Optimizer(model, phi, params, timing=False)
    for _ in range(W):
        opt.step()

    def barrier():
        if world > 1:
            dist.barrier()

    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    fem.PCG_PROFILE = []
    launches0 = lib.lsg_launch_count()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    recs = [opt.step() for _ in range(K)]
    e1.record(stream)
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    launches = lib.lsg_launch_count() - launches0
    prof, fem.PCG_PROFILE = fem.PCG_PROFILE, None
    t_local = e0.elapsed_time(e1) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return {"mesh": mesh, "model": opt.model, "opt": opt, "recs": recs, "prof": prof,
            "t_local": t_local, "t_max": float(t.item()), "launches": int(launches)}


def pcg_roofline(lw, hbm, peak_kind, ncu):
    from paper_2601_05709_b200 import _lib

    mesh = lw["mesh"]
    d, N, E = mesh.dim, mesh.num_vertices, mesh.num_elements
    prof = lw["prof"]
    state = [p for p in prof if p["kind"] == _lib.LSG_OP_ELASTICITY]
    pcg_ms = sum(p["events"][0].elapsed_time(p["events"][1]) for p in state)
    rhs_iters = sum(p["rhs_iters"] for p in state)
    launched = sum(p["launched"] for p in state)
    max_iters = sum(p["max_iters"] for p in state)
    # (80 k + 16) d N + E bytes per iteration of k right-hand sides
    # = 80 d N per right-hand-side iteration + (16 d N + E) per batched iteration
    pcg_bytes = 80.0 * d * N * rhs_iters + (16.0 * d * N + E) * max_iters
    achieved = pcg_bytes / (pcg_ms / 1e3) / 1e9 if pcg_ms > 0 else 0.0
    all_ms = sum(p["events"][0].elapsed_time(p["events"][1]) for p in prof)
    kern = dict(ncu.get(f"pcg{d}d", {}))
    traffic = kern.get("dram_bytes_per_iteration")
    launches = ncu.get("pcg_cfg5" if d == 3 else "pcg_cfg2", {}).get("launches", [])
    if launches:  # per-launch split of one batched iteration (ncu, cold, serialised)
        kern["split_us"] = [[r["kernel"].split("(")[0].replace("void ", ""), round(r.get("us", 0.0), 1),
                             round((r.get("dram_read", 0.0) + r.get("dram_write", 0.0)) / 1e6, 1)]
                            for r in launches]
    return {"bound": "hbm", "kernel": PCG_KERNELS[d], "achieved": achieved, "peak": hbm, "unit": "GB/s",
            "frac": achieved / hbm, "traffic": traffic, "peak_kind": peak_kind,
            "bytes_per_iteration": "(80k+16) d N + E per k-rhs iteration (canonical two-pass)",
            "us_per_batched_iteration": pcg_ms * 1e3 / max(max_iters, 1),
            "pcg_ms_in_timed_region": pcg_ms, "pcg_share_of_step": all_ms / (lw["t_local"] * 1e3),
            "rhs_iterations": rhs_iters, "batched_iterations": max_iters, "launched_iterations": launched,
            "ncu": kern or None,
            "traffic_note": "DRAM bytes per batched PCG iteration (all its launches) from the committed "
                            "ncu --set full capture (profiles/r02_ncu_kernels.json, cold cache)"}


def b200_arm(args, world, rank, local):
    import torch
    import torch.distributed as dist

    import paper_2601_05709_b200 as lsg
    from paper_2601_05709_b200 import configs

    torch.cuda.set_device(local)
    c = configs.case(args.config)
    W, K = args.warmup, args.steps
    sharded = bool(args.shard_loads and world > 1)
    hbm, peak_kind = peaks()
    ncu = ncu_kernels()

    clocks = ClockSampler(local)
    clocks.start()
    lw = loop_window(c, W, K, world, sharded, dist)
    clk = clocks.stop()
    mesh, model, recs = lw["mesh"], lw["model"], lw["recs"]
    d, N, E = mesh.dim, mesh.num_vertices, mesh.num_elements
    k = int(model.load_vectors.shape[0])
    t_max = lw["t_max"]
    value = (1 if sharded else world) * K / t_max
    roof = pcg_roofline(lw, hbm, peak_kind, ncu)
    counts = window_counts(recs)
    launches = lw["launches"]

    # ---- standalone apply of this config's operator (k RHS), L2 flushed ------------------
    op = lw["opt"].model.operator(lw["opt"].phi)
    u = torch.randn((k, d * N), dtype=torch.float64, device="cuda")
    ms = flushed_apply_ms(op, u)
    apply_bytes = 16.0 * d * k * N + E
    apply = {"k": k, "ms": ms, "dof_per_s": k * d * N / (ms / 1e3), "gbs": apply_bytes / (ms / 1e3) / 1e9,
             "frac": apply_bytes / (ms / 1e3) / 1e9 / hbm, "bytes": apply_bytes,
             "flush": "256 MB write + 256 MB read of another buffer before each launch"}
    del op, u
    del lw

    largest = None
    if not args.no_largest and rank == 0:
        largest = largest_applies(hbm, ncu)

    # ---- end to end: the config's own run through the public run() from host buffers ------
    e2e = None
    if not args.no_e2e:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        m0 = configs.build(c)[0]
        phi_host = torch.from_numpy(np.ascontiguousarray(c.phi0(m0.vertices if c.name != "cfg4" else None),
                                                         dtype=np.float64)).pin_memory()
        del m0
        out_host = torch.empty(N, dtype=torch.float64).pin_memory()
        d2h = [0]

        def on_record(rec, phi_dev):
            out_host.copy_(phi_dev.values, non_blocking=False)
            d2h[0] += N * 8 + 8 * 8

        torch.cuda.synchronize()
        t0 = time.perf_counter()
        m2, model2, _, params2 = configs.build(c)             # loads assembled host-side, uploaded
        loads_host = model2.load_vectors.cpu().pin_memory()
        model2._loads.copy_(loads_host, non_blocking=True)    # explicit pinned H2D of the loads
        phi_dev = lsg.LevelSetField.from_field(
            lsg.FemField(lsg.FunctionSpace(m2, 1), phi_host.to("cuda", non_blocking=True)))
        _, hist = lsg.run(model2, phi_dev, params2, on_record=on_record, timing=False)
        torch.cuda.synchronize()
        t_e2e = time.perf_counter() - t0
        te = torch.tensor([t_e2e], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(te, op=dist.ReduceOp.MAX)
        n_it = len(hist)
        h2d = (phi_host.numel() + loads_host.numel()) * 8
        e2e = {"value": world * n_it / float(te.item()), "unit": "iters/s",
               "h2d_bytes_per_step": int(h2d / n_it), "d2h_bytes_per_step": int(d2h[0] / n_it),
               "iterations": n_it, "time_to_solution_s": float(te.item()),
               "final": {"J": hist[-1].cost, "C": float(hist[-1].constraint[0])},
               "note": f"time to solution: the config's own {n_it}-iteration run through the public "
                       "run() from pinned host phi0 / loads (cold start, mesh + model setup included), "
                       "phi + record read back to the host every iteration"}
        del model2, phi_dev

    # ---- secondary: the 2D bridge loop (BASELINE configs[1]) --------------------------------
    secondary = None
    if not args.no_secondary and args.config != "cfg2" and rank == 0 and world == 1:
        c2 = configs.case("cfg2")
        lw2 = loop_window(c2, 3, 10, 1, False, dist)
        roof2 = pcg_roofline(lw2, hbm, peak_kind, ncu)
        secondary = {"config": WORKLOAD["cfg2"], "window": "warmup 3, 10 timed iterations",
                     "value": 10 / lw2["t_max"], "unit": "iters/s",
                     "pcg_us_per_iteration": roof2["us_per_batched_iteration"],
                     "pcg_frac": roof2["frac"], "pcg_share_of_step": roof2["pcg_share_of_step"],
                     "rhs_pcg_iters_per_outer": window_counts(lw2["recs"])["rhs_pcg_iters"]}
        del lw2

    # ---- CPU baseline (rank 0, N = 1 only) ------------------------------------------------
    cpu = None
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        t0 = time.perf_counter()
        units = cpu_units(c, procs=1)
        t_sample = time.perf_counter() - t0
        s_it = cpu_seconds_per_iteration(units, counts)
        cpu = {"value": 1.0 / s_it, "unit": "iters/s", "cores": 1, "kind": "port",
               "extrapolated_s_per_iteration": s_it, "units": units, "counts": counts,
               "apply_dof_per_s": None,
               "sample": f"oracle (numpy/scipy restatement of the reference path) on a {units['slab']} "
                         f"slab of {args.config} (x{units['scale']:.0f} to the full mesh), 1 core, "
                         f"{t_sample:.1f} s of CPU work: assembly + elimination, scipy-cg Jacobi-PCG "
                         "iterations, S1 + derivative vector, H1 velocity CG iterations, transport and "
                         "reinit substeps; extrapolated to one outer iteration with the counts this "
                         "run's timed window measured"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "iters/s", "n_gpus": world, "steps": K,
            "warmup": W, "ms_per_step": 1e3 * t_max / K, "higher_is_better": True,
            "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic",
            "config": {"workload": f"{WORKLOAD[args.config]}, full loop (state PCG rtol 1e-10, S1+RHS, "
                                   f"H1 CG, transport, reinit every {c.reinit_step})",
                       "window": f"iterations {W}..{W + K - 1} of the run (after {W} untimed warm-up "
                                 "iterations); the PCG work per iteration depends on the window",
                       "nodes": N, "elements": E, "load_cases": k,
                       "l2": "PCG working set exceeds the 126 MB L2 (cfg5: ~1.4 GB); standalone apply "
                             "timings flush L2 before each launch",
                       "parallelism": (f"load cases sharded over {world} GPUs" if sharded else
                                       f"replicas x{world}" if world > 1 else "single GPU")},
            "roofline": roof,
            "apply": apply,
            "apply_largest": largest,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "secondary": secondary,
            "gpu_launches": launches,
            "clocks": clk,
            "history": {"J": [r.cost for r in recs], "C": [float(r.constraint[0]) for r in recs],
                        "counts_per_outer": counts,
                        "cg_iters": [list(r.cg_iters) for r in recs],
                        "velocity_iters": [r.velocity_iters for r in recs]},
        }
        print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# Reference arm: the reference's CPU algorithm (the oracle port) on the host cores
# ---------------------------------------------------------------------------------------------

def reference_arm(args, world, rank, local):
    """Each step: one bounded sample of the workload (per-unit costs on a slab of the
    config's mesh), extrapolated to one outer iteration with the per-iteration counts
    the B200 arm measured in the same window (profiles/r02_calibration.json)."""
    if rank != 0:
        return
    from paper_2601_05709_b200 import configs

    c = configs.case(args.config)
    procs = min(os.cpu_count() or 1, 8)
    cal = None
    try:
        with open(CALIBRATION) as f:
            cal_all = json.load(f)
        window = f"w{args.warmup}k{args.steps}"
        entry = cal_all.get(args.config, {})
        cal = entry.get(window) or (entry[sorted(entry)[0]] if entry else None)
        cal_window = window if window in entry else (sorted(entry)[0] if entry else None)
    except Exception:
        cal_window = None
    if cal is None:
        print(json.dumps({"impl": "reference", "unavailable": f"no calibration for {args.config} in "
                                                              "profiles/r02_calibration.json"}))
        return
    per_step, samples = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        units = cpu_units(c, procs=procs)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            per_step.append(dt)
            samples.append(cpu_seconds_per_iteration(units, cal))
    s_it = statistics.median(samples)
    v = 1.0 / s_it
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(per_step),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        "config": {"workload": f"{WORKLOAD[args.config]} (same as the b200 arm)"},
        "extrapolation": {"s_per_outer_iteration": s_it, "counts_per_outer": cal,
                          "counts_window": cal_window, "units_last_step": units,
                          "note": "value = 1 / s_per_outer_iteration; each step measured the per-unit "
                                  "costs on a slab and extrapolated; ms_per_step is the step's real "
                                  "duration"},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": units["pcg_procs"], "kind": "port",
                         "sample": f"per step: oracle (numpy/scipy restatement of the reference) on a "
                                   f"{units['slab']} slab of {args.config}, scaled x{units['scale']:.0f}: "
                                   f"assembly + elimination, scipy-cg PCG iterations ({units['pcg_procs']} "
                                   "load cases in parallel processes), S1 + derivative vector, H1 velocity "
                                   "CG iterations, transport + reinit substeps"},
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

"""bench.py's reference arm prints one JSON line with the driver's contract keys
(CPU only: the arm times the oracle port on the host; a small config keeps it fast)."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    res = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "cfg1", "--steps", "1", "--warmup", "0"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert res.returncode == 0, res.stderr[-2000:]
    line = json.loads(res.stdout.strip().splitlines()[-1])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "cpu_baseline", "e2e"):
        assert key in line, key
    assert line["impl"] == "reference" and line["value"] > 0 and line["higher_is_better"] is True
    assert line["cpu_baseline"]["kind"] == "port" and line["cpu_baseline"]["cores"] >= 1
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["value"] == line["value"]


def test_cpu_sampler_units_and_extrapolation():
    """The CPU arm's slab sampler returns positive per-unit costs scaled to the full mesh,
    and the extrapolation is the documented linear combination with the counts."""
    import sys
    sys.path.insert(0, ROOT)
    import bench
    from paper_2601_05709_b200 import configs
    c = configs.case("cfg1")
    u = bench.cpu_units(c, procs=1, slab=4)
    assert u["scale"] == 80 / 4 and u["slab"] == "160x4"
    for key in ("assembly_s", "pcg_rhs_iter_s", "s1_rhs_s", "velocity_iter_s", "transport_substep_s",
                "reinit_substep_s"):
        assert u[key] > 0.0, key
    counts = {"rhs_pcg_iters": 100.0, "velocity_iters": 10.0, "transport_substeps": 5.0, "reinit_substeps": 2.0}
    s = bench.cpu_seconds_per_iteration(u, counts)
    want = (u["assembly_s"] + 100 * u["pcg_rhs_iter_s"] + u["s1_rhs_s"] + 10 * u["velocity_iter_s"]
            + 5 * u["transport_substep_s"] + 2 * u["reinit_substep_s"])
    assert abs(s - want) <= 1e-12 * want


def test_calibration_covers_the_bench_configs_and_windows():
    import json
    cal = json.load(open(os.path.join(ROOT, "profiles", "r02_calibration.json")))
    for name in ("cfg1", "cfg2", "cfg3", "cfg5"):
        for window in ("w5k20", "w3k10"):
            counts = cal[name][window]
            assert counts["rhs_pcg_iters"] > 0 and counts["velocity_iters"] > 0
            assert set(counts) == {"rhs_pcg_iters", "velocity_iters", "transport_substeps", "reinit_substeps"}

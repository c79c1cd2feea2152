#!/usr/bin/env python
"""Summarise the round's ncu --set full captures (tools/ncu_extract.sh *_raw.csv) into
profiles/r02_ncu_kernels.json, the file bench.py reads for `traffic` and the fp64-pipe
evidence.

    python tools/ncu_kernels_json.py gpurun_out > profiles/r02_ncu_kernels.json
"""
import csv
import json
import os
import sys

UNIT = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
        "msecond": 1e-3, "second": 1.0, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}
METRICS = {
    "us": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "fp64_pipe_pct": "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "warp_instructions": "smsp__inst_executed.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "local_loads": "smsp__sass_inst_executed_op_local_ld.sum",
}
STALLS = "smsp__average_warps_issue_stalled_"


def rows(path):
    r = list(csv.reader(open(path)))
    return r[0], r[1], r[2:]


def launch_record(h, units, row):
    out = {"kernel": row[h.index("Kernel Name")]}
    for key, m in METRICS.items():
        if m in h:
            i = h.index(m)
            try:
                v = float(row[i].replace(",", ""))
            except ValueError:
                continue
            scale = UNIT.get(units[i], 1.0)
            if key == "us":
                v = v * scale * 1e6
            elif key.startswith("dram_") and key != "dram_pct":
                v = v * scale
            out[key] = v
    stalls = {}
    for i, name in enumerate(h):
        if name.startswith(STALLS) and name.endswith("_per_issue_active.ratio"):
            try:
                stalls[name[len(STALLS):-len("_per_issue_active.ratio")]] = float(row[i])
            except ValueError:
                pass
    if stalls:
        out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:8])
    return out


def main(d):
    out = {"source": "ncu --set full --clock-control none (cold cache, serialised launches), "
                     "tools/gpu_profile_r02.sh; per-launch records"}
    for name in sorted(os.listdir(d)):
        if not name.endswith("_raw.csv"):
            continue
        h, units, body = rows(os.path.join(d, name))
        recs = [launch_record(h, units, r) for r in body if r and r[0]]
        key = name[len("r02_"):-len("_raw.csv")] if name.startswith("r02_") else name[:-8]
        out[key] = {"launches": recs}
    # one batched PCG iteration = every captured launch of the pcg captures
    for key in [k for k in out if k.startswith("pcg_")]:
        recs = out[key]["launches"]
        out[key]["dram_bytes_per_iteration"] = sum(r.get("dram_read", 0) + r.get("dram_write", 0) for r in recs)
        out[key]["us_serialised_per_iteration"] = sum(r.get("us", 0) for r in recs)
    if "pcg_cfg5" in out:
        out["pcg3d"] = {k: out["pcg_cfg5"][k] for k in ("dram_bytes_per_iteration", "us_serialised_per_iteration")}
    if "pcg_cfg2" in out:
        out["pcg2d"] = {k: out["pcg_cfg2"][k] for k in ("dram_bytes_per_iteration", "us_serialised_per_iteration")}
    for c in ("cfg4", "cfg5"):
        if f"apply_{c}" in out and out[f"apply_{c}"]["launches"]:
            r = out[f"apply_{c}"]["launches"][0]
            out[f"apply_{c}"].update({"dram_bytes": r.get("dram_read", 0) + r.get("dram_write", 0),
                                      "fp64_pipe_pct": r.get("fp64_pipe_pct"), "us": r.get("us")})
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])

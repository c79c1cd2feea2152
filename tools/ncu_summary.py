#!/usr/bin/env python
"""Summarise ncu output for profiles/: per-kernel duration, DRAM bytes, throughput,
occupancy and top stall reasons (from a --set full report), or launch shares (from a
--metrics gpu__time_duration.sum --csv launch list).

    python tools/ncu_summary.py report.ncu-rep        # full-set report
    python tools/ncu_summary.py launches.csv          # launch list
"""

import collections
import csv
import io
import subprocess
import sys

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__grid_size", "launch__block_size",
       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum"]


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = collections.defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki].split("(")[0][:70]].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'share':>6} {'n':>5} {'mean_us':>9}  kernel   (cold-cache, serialised; total {tot/1e3:.1f} us)")
    for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        print(f"{100*sum(v)/tot:5.1f}% {len(v):5d} {sum(v)/len(v)/1e3:9.2f}  {k}")


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units = rows[0], rows[1]
    name = h.index("Kernel Name")
    for r in rows[2:]:
        print(f"== {r[name].split('(')[0]}")
        for m in RAW:
            if m in h:
                i = h.index(m)
                print(f"   {m:60s} {r[i]:>14s} {units[i]}")
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    seen = set()
    for r in csv.reader(io.StringIO(det)):
        if len(r) > 14 and r[12] in ("Warp Cycles Per Issued Instruction", "Achieved Occupancy",
                                     "Theoretical Occupancy", "DRAM Throughput", "Duration"):
            key = (r[4].split("(")[0], r[12])
            if key not in seen:
                seen.add(key)
                print(f"   {key[0][:40]:40s} {r[12]:40s} {r[14]:>10s} {r[13]}")


if __name__ == "__main__":
    p = sys.argv[1]
    launches(p) if p.endswith(".csv") else full(p)

#!/usr/bin/env python
"""Per-opcode dynamic instruction counts and stall samples of one kernel in an
ncu --set full report (source page, SASS view).

    python tools/ncu_ops.py report.ncu-rep [top]
"""
import collections
import csv
import io
import re
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, isrc, ismp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot, stot = 0, 0
ops, samp = collections.Counter(), collections.Counter()
for r in rows[2:]:
    try:
        n = int(r[ie])
    except (ValueError, IndexError):
        continue
    op = re.sub(r"^@!?U?P\w+\s+", "", r[isrc].strip()).split(" ")[0].split(".")[0]
    tot += n
    ops[op] += n
    s = int(r[ismp] or 0)
    samp[op] += s
    stot += s
print(f"total warp instructions {tot}, stall samples {stot}")
for k, v in ops.most_common(top):
    print(f"{k:12s} {v:12d} {v / tot * 100:5.1f}%   samples {samp[k] / max(stot, 1) * 100:5.1f}%")

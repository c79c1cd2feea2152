#!/usr/bin/env python
"""Attribute an ncu report's per-SASS execution counts to CUDA source lines.

    python tools/sass_lines.py report.ncu-rep obj.o kernel_mangled_name [top]

Disassembles the object's cubin with line info (nvdisasm -g), maps every
instruction offset to its innermost source line, and joins with the ncu SASS
execution counts (same instruction order).
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, fn = sys.argv[1:4]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
cub = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cub)], capture_output=True, text=True).stdout.splitlines()
start = next(i for i, l in enumerate(dis) if l.startswith(fn + ":"))
lines, cur = [], None
for l in dis[start + 1:]:
    if l.startswith("\t.section") or (l and not l[0].isspace() and l.endswith(":") and not l.startswith(".")):
        if lines and l.startswith("\t.section"):
            break
    m = re.search(r'//## File "([^"]+)", line (\d+)', l)
    if m:
        cur = f"{os.path.basename(m.group(1))}:{m.group(2)}"
        continue
    if re.match(r"\s+/\*[0-9a-f]+\*/\s+\S", l):
        lines.append((cur, l.split("*/", 1)[1].strip()))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie = h.index("Instructions Executed")
counts = [int(r[ie]) for r in rows[2:] if len(r) > ie and r[ie].isdigit()]
agg = collections.Counter()
for (src, _), n in zip(lines, counts):
    agg[src] += n
tot = sum(counts)
print(f"sass {len(lines)} ncu {len(counts)} total {tot}")
for k, v in agg.most_common(top):
    print(f"{v:11d} {v / tot * 100:5.1f}%  {k}")

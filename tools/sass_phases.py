#!/usr/bin/env python
"""Split an ncu SASS source export (--page source --csv --print-source sass) at BAR
instructions and report per-segment stall samples and instruction counts.
usage: ncu -i rep --page source --csv --print-source sass > s.csv; python tools/sass_phases.py s.csv"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ii, ex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
segs, cur = [], {"samples": 0, "inst": 0, "ops": Counter(), "first": None}
total = 0
for r in rows[2:]:
    if len(r) <= ex:
        continue
    src = r[si].strip()
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    s = int(float(r[ii] or 0)); n = int(float(r[ex] or 0))
    total += s
    cur["samples"] += s; cur["inst"] += n; cur["ops"][op.split(".")[0]] += n
    if cur["first"] is None:
        cur["first"] = r[0]
    if op.startswith("BAR"):
        segs.append(cur); cur = {"samples": 0, "inst": 0, "ops": Counter(), "first": None}
segs.append(cur)
for i, sg in enumerate(segs):
    if sg["inst"] == 0:
        continue
    top = ", ".join(f"{k}:{v}" for k, v in sg["ops"].most_common(6))
    print(f"seg {i:2d} @{sg['first']}: samples {sg['samples']:7d} ({100*sg['samples']/max(total,1):5.1f}%) inst {sg['inst']:10d}  {top}")

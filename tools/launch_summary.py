#!/usr/bin/env python
"""Summarise an ncu --metrics gpu__time_duration.sum --csv launch list: count, mean, share per kernel.
usage: python tools/launch_summary.py launches.csv "<header line>" """
import csv, sys
from collections import defaultdict
rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if not l.startswith("=="))]
h = rows[0]
ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
t = defaultdict(list)
for r in rows[1:]:
    if len(r) > vi and r[mi] == "gpu__time_duration.sum":
        t[r[ki]].append(float(r[vi].replace(",", "")))
tot = sum(sum(v) for v in t.values())
print(sys.argv[2] if len(sys.argv) > 2 else sys.argv[1])
print("count  mean_ns  share  kernel")
for k, v in sorted(t.items(), key=lambda kv: -sum(kv[1])):
    print(f"{len(v):5d} {sum(v) / len(v):11.0f} {100 * sum(v) / tot:5.1f}%  {k[:80]}")

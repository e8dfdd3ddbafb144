#!/usr/bin/env python
"""Per-segment (split at BAR) stall-reason breakdown of an ncu SASS source export.
usage: python tools/sass_stalls.py s.csv"""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ex = h.index("Source"), h.index("Instructions Executed")
st = [i for i, c in enumerate(h) if c.startswith("stall_")]
segs, cur = [], Counter()
tot = Counter()
for r in rows[2:]:
    if len(r) <= ex:
        continue
    src = r[si].strip()
    for i in st:
        v = int(float(r[i] or 0)); cur[h[i][6:]] += v; tot[h[i][6:]] += v
    op = src.split()[0] if src else ""
    if op.startswith("@"):
        op = src.split()[1]
    if op.startswith("BAR"):
        segs.append(cur); cur = Counter()
segs.append(cur)
T = sum(tot.values())
for k, sg in enumerate(segs):
    s = sum(sg.values())
    if s == 0:
        continue
    print(f"seg {k:2d} {100*s/T:5.1f}%  " + ", ".join(f"{a}:{100*b/T:.1f}" for a, b in sg.most_common(5)))
print("total", ", ".join(f"{a}:{100*b/T:.1f}" for a, b in tot.most_common(10)))

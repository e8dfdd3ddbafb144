#!/usr/bin/env python
"""Top stall instructions of one BAR-delimited segment of an ncu SASS export.
usage: python tools/sass_top.py s.csv SEG [N]"""
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
seg, topn = int(sys.argv[2]), int(sys.argv[3]) if len(sys.argv) > 3 else 15
h = rows[1]; si = h.index("Source"); ii = h.index("Warp Stall Sampling (All Samples)"); ex = h.index("Instructions Executed")
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
cur, out = 0, []
for n, r in enumerate(rows[2:]):
    if len(r) <= ex:
        continue
    if cur == seg:
        st = sorted(((float(r[c] or 0), h[c][6:]) for c in sc), reverse=True)[:3]
        out.append((int(float(r[ii] or 0)), n, int(float(r[ex] or 0)), r[si][:60], [(int(a), b) for a, b in st if a > 0]))
    if r[si].strip().split()[0:1] and ("BAR" in r[si].split()[0] or (r[si].startswith("@") and "BAR" in r[si])):
        cur += 1
out.sort(reverse=True)
for o in out[:topn]:
    print(o)

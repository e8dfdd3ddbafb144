import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
si, ex = h.index("Source"), h.index("Instructions Executed")
wf = h.index("L1 Wavefronts Shared"); wfi = h.index("L1 Wavefronts Shared Ideal")
l2 = h.index("L2 Theoretical Sectors Global")
segs=[]; cur=[0,0,0,0]
for r in rows[2:]:
    if len(r)<=ex: continue
    src=r[si].strip(); op=src.split()[0] if src else ""
    if op.startswith("@"): op=src.split()[1]
    f=lambda i: int(float(r[i] or 0))
    cur[0]+=f(wf); cur[1]+=f(wfi); cur[2]+=f(l2); cur[3]+=f(ex)
    if op.startswith("BAR"): segs.append(cur); cur=[0,0,0,0]
segs.append(cur)
T=sum(s[0] for s in segs)
for k,s in enumerate(segs):
    if s[3]: print(f"seg {k:2d} wf {s[0]:10d} ({100*s[0]/T:4.1f}%) ideal {s[1]:10d} l2sect {s[2]:9d} inst {s[3]}")

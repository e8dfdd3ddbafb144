timeout 300 python bench.py --no-cpu-baseline --redraw --steps 1 --warmup 3 --batch 256 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_zf_warp -s 3 -c 1 -o /tmp/zfw -f python bench.py --no-cpu-baseline --redraw --steps 1 --warmup 3 --batch 256 > gpurun_out/ncu_zfw.log 2>&1
python tools/ncu_summary.py /tmp/zfw.ncu-rep > gpurun_out/zfw_summary.txt 2>&1
ncu -i /tmp/zfw.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/zfw.csv
python - > gpurun_out/zfw_top.txt <<'PY'
import csv
rows=list(csv.reader(open('/tmp/zfw.csv'))); h=rows[1]
si=h.index("Source"); ex=h.index("Instructions Executed"); sm=h.index("Warp Stall Sampling (All Samples)")
L=[(int(float(r[sm] or 0)), i, int(float(r[ex] or 0)), r[si][:80]) for i,r in enumerate(rows[2:]) if len(r)>ex]
tot=sum(x[0] for x in L)
for x in sorted(L,reverse=True)[:25]: print(round(100*x[0]/tot,1), x[1:])
# cumulative by region of 100 instructions
import collections
c=collections.Counter()
for x in L: c[x[1]//100]+=x[0]
print([(k*100, round(100*v/tot,1)) for k,v in sorted(c.items())])
PY

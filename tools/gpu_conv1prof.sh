python tools/cnn_one.py C5 64 >/dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tc -s 0 -c 1 -o /tmp/c1 -f python tools/cnn_one.py C5 64 > gpurun_out/ncu_c1.log 2>&1
ncu -i /tmp/c1.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/c1.csv
python - > gpurun_out/c1_top.txt <<'PY'
import csv, collections
rows=list(csv.reader(open('/tmp/c1.csv'))); h=rows[1]
si=h.index("Source"); ex=h.index("Instructions Executed"); sm=h.index("Warp Stall Sampling (All Samples)")
L=[(int(float(r[sm] or 0)), i, int(float(r[ex] or 0)), r[si][:80]) for i,r in enumerate(rows[2:]) if len(r)>ex]
tot=sum(x[0] for x in L)
for x in sorted(L,reverse=True)[:30]: print(round(100*x[0]/tot,1), x[1:])
c=collections.Counter()
for x in L: c[x[1]//50]+=x[0]
print([(k*50, round(100*v/tot,1)) for k,v in sorted(c.items()) if v])
PY

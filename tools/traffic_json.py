#!/usr/bin/env python
"""Write profiles/traffic_<cfg>.json (DRAM bytes per launch of the step's kernels) from the
raw CSV page of an ncu --set full capture of `bench.py --steps 1 --warmup 3` (the bench
launch configuration).  usage: python tools/traffic_json.py raw.csv C2 1024 profiles/traffic_c2.json SOURCE"""
import csv
import json
import sys

SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
raw, cfg, batch, out, source = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4], sys.argv[5]
rows = list(csv.reader(open(raw)))
h, units = rows[0], rows[1]
ik, ir, iw = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
roles = {"fdcnn": ("k_cnn_fused", "k_conv"), "chain_txrx": ("k_chain_tx", "k_chain_cl"),
         "combine": ("k_rx_combine",), "precode": ("k_precode",)}
res = {}
for r in rows[2:]:
    if len(r) != len(h):
        continue
    name = r[ik]
    for role, keys in roles.items():
        if any(k in name for k in keys) and role not in res:
            rd = float(r[ir]) * SCALE[units[ir]]
            wr = float(r[iw]) * SCALE[units[iw]]
            res[role] = {"kernel": name[:60], "dram_read_bytes": rd, "dram_write_bytes": wr,
                         "bytes_per_launch": rd + wr, "config": cfg, "batch": batch, "source": source}
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res, indent=1))

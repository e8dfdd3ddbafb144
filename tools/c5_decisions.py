"""Diagnostic: decision parity at a large config (one symbol vs the oracle)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import fdpd_oracle as O
from paper_2205_05158_b200.chain import Chain, Shapes
from workload import configs, gen

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.get(name)
inp = gen.make_inputs(cfg, range(8))
ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=8)
s = torch.from_numpy(inp["s"]).cuda(); idx = torch.from_numpy(inp["idx"].astype(np.int32)).cuda().to(torch.uint16)
dec = torch.zeros(idx.shape, dtype=torch.uint16, device="cuda")
yhat, counts, _ = ch.step(s, idx, dec=dec)
torch.cuda.synchronize()
o = O.run_config(cfg, gen.make_inputs(cfg, [5]))
g = yhat.cpu().numpy()[5:6].astype(np.complex128); d = dec.cpu().numpy()[5:6]
zo, zg = o["yhat"] / o["alpha"], g / ch.alpha
c = 1 / np.sqrt(2 * (cfg.M_qam - 1) / 3)
err = np.abs(zg - zo)
print("yhat rel", np.linalg.norm(g - o["yhat"]) / np.linalg.norm(o["yhat"]))
print("|z| rms", np.sqrt(np.mean(abs(zo) ** 2)), "median", np.median(abs(zo)), "abs err max", err.max(), "median", np.median(err))
mm = d != o["dec"]
print("mismatches", int(mm.sum()), "of", d.size)
for v in (zo.real / c, zo.imag / c):
    dist = np.abs(v - 2 * np.round(v / 2)) * c
    print(" axis dist-to-boundary of mismatches (unit-energy units):", np.sort(dist[mm])[:10], "err there", err[mm][:10])

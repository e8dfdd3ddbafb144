#!/usr/bin/env python
"""Determinism / parity check of the tensor-core GMP at a full bench batch: chain_txrx_pre twice
(tensor cores) and once (SIMT) on the same precoded spectra; reports the (symbol, antenna) rows
that differ between repeats and the worst relative error against the SIMT path."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from workload import configs, gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
cfg = configs.get(name)
inp = gen.make_inputs(cfg, range(n))
dev = "cuda"
h_fd, P, alpha = fdpd.zf_precoder_build(torch.from_numpy(inp["h_taps"]).to(dev), cfg.N_ifft, cfg.N_d, cfg.rho)
X = fdpd.precode(P, torch.from_numpy(inp["s"]).to(dev))
coef = torch.from_numpy(inp["coef"]).to(dev)
outs = []
for path in (2, 2, 2, 1):
    fdpd.set_gmp_path(path)
    y, XPA = fdpd.chain_txrx_pre(X, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    torch.cuda.synchronize()
    outs.append((y.clone(), XPA.clone()))
for r in (1, 2):
    d = (outs[0][0].view(torch.int64) != outs[r][0].view(torch.int64)).any(dim=-1)
    bad = torch.nonzero(d).tolist()
    print(f"repeat {r}: rows differing {len(bad)} of {n * cfg.B}: {bad[:12]}")
    if bad:
        i, b = bad[0]
        a, c = outs[0][0][i, b], outs[r][0][i, b]
        idx = torch.nonzero(a.view(torch.int64) != c.view(torch.int64)).flatten()
        print("   first differing samples", idx[:20].tolist(), "of", idx.numel())
ys, yt = outs[3][0], outs[0][0]
num = (ys - yt).abs().pow(2).sum(dim=-1).sqrt()
den = ys.abs().pow(2).sum(dim=-1).sqrt()
r = (num / den).flatten()
print("rel vs SIMT per row: max", float(r.max()), "median", float(r.median()), "rows > 1e-5:", int((r > 1e-5).sum()))

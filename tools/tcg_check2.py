#!/usr/bin/env python
"""Tensor-core GMP: the same symbols through chain_txrx_pre in one 32-symbol launch and in
launches of 8 / 16 symbols (the native runtime's chunking), plus the SIMT path; reports rows
that differ."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from workload import configs, gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
n = 32
cfg = configs.get(name)
inp = gen.make_inputs(cfg, range(n))
dev = "cuda"
h_fd, P, alpha = fdpd.zf_precoder_build(torch.from_numpy(inp["h_taps"]).to(dev), cfg.N_ifft, cfg.N_d, cfg.rho)
X = fdpd.precode(P, torch.from_numpy(inp["s"]).to(dev))
coef = torch.from_numpy(inp["coef"]).to(dev)


def run(path, chunk):
    fdpd.set_gmp_path(path)
    y = torch.empty((n, cfg.B, cfg.N_ifft), dtype=torch.complex64, device=dev)
    XPA = torch.empty((n, cfg.B, cfg.N_d), dtype=torch.complex64, device=dev)
    for s0 in range(0, n, chunk):
        fdpd.chain_txrx_pre(X[s0:s0 + chunk], coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft, y=y[s0:s0 + chunk],
                            XPA=XPA[s0:s0 + chunk])
    torch.cuda.synchronize()
    return y


ref = run(2, 32)
for chunk in (8, 16, 1, 32):
    y = run(2, chunk)
    d = (ref.view(torch.int64) != y.view(torch.int64)).any(dim=-1)
    bad = torch.nonzero(d).tolist()
    print(f"tc chunk {chunk}: rows differing {len(bad)}: {bad[:10]}", flush=True)
ys = run(1, 8)
r = ((ys - ref).abs().pow(2).sum(-1).sqrt() / ys.abs().pow(2).sum(-1).sqrt()).flatten()
print("tc vs simt max rel", float(r.max()))

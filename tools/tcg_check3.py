#!/usr/bin/env python
"""Tensor-core GMP chain after shared memory was poisoned with different patterns, and after a
tensor-core precode: bitwise comparison of y (uninitialised-read / cross-kernel interaction hunt)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from workload import configs, gen  # noqa: E402

cfg = configs.get(sys.argv[1] if len(sys.argv) > 1 else "C5")
n = 32
inp = gen.make_inputs(cfg, range(n))
dev = "cuda"
h_fd, P, alpha = fdpd.zf_precoder_build(torch.from_numpy(inp["h_taps"]).to(dev), cfg.N_ifft, cfg.N_d, cfg.rho)
s = torch.from_numpy(inp["s"]).to(dev)
Ppk = fdpd.precode_pack(P)
X = fdpd.precode_packed(Ppk, s, math=fdpd.MATH_FP32_TC)
coef = torch.from_numpy(inp["coef"]).to(dev)
fdpd.set_gmp_path(2)


def chain():
    y, XPA = fdpd.chain_txrx_pre(X, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    torch.cuda.synchronize()
    return y.clone(), XPA.clone()


ref = chain()
for tag, pre in (("plain", lambda: None), ("poison 0", lambda: fdpd.debug_poison_smem(0)),
                 ("poison nan", lambda: fdpd.debug_poison_smem(0x7FC0DEAD)),
                 ("poison big", lambda: fdpd.debug_poison_smem(0x4E6E6B28)),
                 ("precode_tc", lambda: fdpd.precode_packed(Ppk, s, math=fdpd.MATH_FP32_TC))):
    for rep in range(2):
        pre()
        y, XPA = chain()
        d = (ref[0].view(torch.int64) != y.view(torch.int64)).any(dim=-1)
        bad = torch.nonzero(d).tolist()
        dx = (ref[1].view(torch.int64) != XPA.view(torch.int64)).any(dim=-1).sum().item()
        print(f"{tag} rep {rep}: y rows differing {len(bad)} {bad[:6]}, XPA rows differing {dx}", flush=True)
        if bad:
            i, b = bad[0]
            idx = torch.nonzero(ref[0][i, b].view(torch.int64) != y[i, b].view(torch.int64)).flatten()
            print("    samples", idx[:16].tolist(), "count", idx.numel(),
                  "max |diff|", float((ref[0][i, b] - y[i, b]).abs().max()), flush=True)

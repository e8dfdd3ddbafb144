#!/usr/bin/env python
"""Phase timeline of the cluster chain kernel (a -DFD_TRACE build: tools/build_variant.sh
variants/libfdpd_trace.so "-DFD_TRACE=1" chain_cl.cu; run with FDPD_LIB=variants/libfdpd_trace.so).
Per CTA: %globaltimer at start / after the X load / after the local IDFT / GMP start / GMP end /
after the cluster barrier / end, and the SM id.  Prints phase durations and, per SM, how the GMP
phases of the two resident CTAs overlap."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from workload import configs, gen  # noqa: E402

cfg = configs.get("C5")
n = 32
inp = gen.make_inputs(cfg, range(n))
dev = "cuda"
rng = np.random.default_rng(1)
X = torch.from_numpy((0.05 * (rng.standard_normal((n, cfg.B, cfg.N_d)) + 1j * rng.standard_normal((n, cfg.B, cfg.N_d)))).astype(np.complex64)).to(dev)
coef = torch.from_numpy(inp["coef"]).to(dev)
for _ in range(3):
    y, XPA = fdpd.chain_txrx_pre(X, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
torch.cuda.synchronize()
nb = 2 * n * cfg.B
buf = np.zeros(65536 * 8, np.uint64)
lib = fdpd.lib()
lib.fd_debug_trace_read.argtypes = [C.c_void_p, C.c_size_t]
assert lib.fd_debug_trace_read(buf.ctypes.data, buf.nbytes) == 0
t = buf.reshape(-1, 8)[:min(nb, 65536)].astype(np.int64)
sm = t[:, 7]
t0 = t[:, 0].min()
names = ["X load", "local IDFT", "combine+relayout", "GMP", "cluster wait", "receive DFT"]
d = np.diff(t[:, :7], axis=1) / 1e3
print("CTAs", len(t), "kernel span %.3f ms" % ((t[:, 6].max() - t0) / 1e6))
for i, nm in enumerate(names):
    print(f"  {nm:18s} mean {d[:, i].mean():7.2f} us  p10 {np.percentile(d[:, i], 10):7.2f}  p90 {np.percentile(d[:, i], 90):7.2f}")
life = (t[:, 6] - t[:, 0]) / 1e3
print("  lifetime           mean %.2f us" % life.mean())
# per SM: fraction of time with 0 / 1 / 2 CTAs in the GMP
tot = np.zeros(3)
for s in np.unique(sm):
    m = sm == s
    ev = [(a, 1) for a in t[m, 3]] + [(b, -1) for b in t[m, 4]]
    ev.sort()
    lo, hi = t[m, 0].min(), t[m, 6].max()
    cur, last = 0, lo
    for tt, dlt in ev:
        tot[min(cur, 2)] += tt - last
        last = tt
        cur += dlt
    tot[min(cur, 2)] += hi - last
print("per-SM time with 0 / 1 / 2 CTAs in the GMP: %.1f %% / %.1f %% / %.1f %%" % tuple(100 * tot / tot.sum()))
# GMP duration vs overlap with the other resident CTA's GMP
ov = np.zeros(len(t))
for s in np.unique(sm):
    idx = np.nonzero(sm == s)[0]
    a, b = t[idx, 3], t[idx, 4]
    for k, i in enumerate(idx):
        o = np.minimum(b, b[k]) - np.maximum(a, a[k])
        o[k] = 0
        ov[i] = np.clip(o, 0, None).sum() / max(b[k] - a[k], 1)
g = d[:, 3]
for lo_, hi_ in ((0, 0.1), (0.1, 0.5), (0.5, 0.9), (0.9, 2)):
    m = (ov >= lo_) & (ov < hi_)
    if m.any():
        print(f"  GMP overlap fraction [{lo_}, {hi_}): {m.sum():6d} CTAs, GMP {g[m].mean():6.2f} us, lifetime {life[m].mean():6.2f} us")
# raw timeline of one SM (first and middle CTAs)
s0 = int(sm[0])
idx = np.nonzero(sm == s0)[0]
idx = idx[np.argsort(t[idx, 0])]
print("SM", s0, "CTAs", len(idx))
for i in list(idx[:8]) + list(idx[100:108]):
    r = (t[i, :7] - t0) / 1e3
    print(f"  cta {i:6d} start {r[0]:8.2f} idft {r[1]:8.2f} comb {r[2]:8.2f} gmp {r[3]:8.2f} .. {r[4]:8.2f} dft {r[5]:8.2f} end {r[6]:8.2f}")

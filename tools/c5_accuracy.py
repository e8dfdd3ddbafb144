"""Diagnostic: end-to-end sensitivity of the C5 PA waveform to the CNN path's rounding.
Runs fdcnn_forward on the SIMT and tensor-core paths for one C5 symbol, then the oracle's
precode -> IDFT -> GMP on each GPU s_tilde, and reports rel-L2 against the all-oracle y."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from oracle import fdpd_oracle as O
from paper_2205_05158_b200 import fdpd
from workload import configs, gen


def rel(a, b):
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = configs.get(name)
sub = gen.make_inputs(cfg, [5])
o = O.run_config(cfg, sub)
s = torch.from_numpy(sub["s"]).cuda()
params = torch.from_numpy(sub["params"]).cuda()
dc = o["s_tilde"].mean(axis=-1, keepdims=True)
for path, code in (("simt", fdpd.CNN_SIMT), ("tensor", fdpd.CNN_TENSOR)):
    fdpd.set_cnn_path(code)
    st = fdpd.fdcnn_forward(params, cfg.chans, s).cpu().numpy().astype(np.complex128)
    err = st - o["s_tilde"]
    y = O.gmp_pa(O.ofdm_modulate(O.precode(o["P"], st), cfg.N_ifft), sub["coef"], cfg.orders, cfg.L, cfg.M)
    print(path, "s_tilde rel", rel(st, o["s_tilde"]), "mean(err)/rms", float(np.sqrt(np.mean(abs(err.mean(-1)) ** 2)) /
          np.sqrt(np.mean(abs(o["s_tilde"]) ** 2))), "-> y rel", rel(y, o["y"]))
fdpd.set_cnn_path(fdpd.CNN_AUTO)

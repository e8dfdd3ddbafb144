#!/usr/bin/env python
"""Small invocations of every kernel family through the C ABI, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck).  Seeded random inputs at tiny sizes that
still take each kernel's real code path (tensor-core CNN layers, cluster-split chain, tensor-core
precode and channel sum, fused / split chains, ZF, impairments, per-symbol redraw, native runtime).
No parity here — tests/ does that; this only has to run every kernel once, cleanly.

usage: compute-sanitizer --tool memcheck python tools/sanitize_cases.py [case ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from paper_2205_05158_b200.chain import Chain, Shapes  # noqa: E402
from workload import configs, gen  # noqa: E402

DEV = "cuda"


def cr(rng, *shape, scale=1.0):
    x = scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))
    return torch.from_numpy(x.astype(np.complex64)).to(DEV)


def step_cfg(cfg, n, **kw):
    inp = gen.make_inputs(cfg, list(range(n)))
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], device=DEV, max_batch=n, **kw)
    s = torch.from_numpy(inp["s"]).to(DEV)
    idx = torch.from_numpy(inp["idx"]).to(DEV)
    dec = torch.zeros(idx.shape, dtype=torch.uint16, device=DEV)
    ch.step(s, idx, dec=dec)
    return ch, inp, s, idx


def case_c1():
    step_cfg(configs.C1, 4)
    ch, inp, s, idx = step_cfg(configs.C1, 4)
    ch.step(s, idx, fused=False)
    taps = torch.from_numpy(gen.channel_taps_per_symbol(configs.C1, list(range(4)))).to(DEV)
    ch.step_redraw(s, idx, taps)


def case_c1_impair():
    cfg = configs.impaired(configs.C1)
    inp = gen.make_inputs(cfg, list(range(4)))
    imp = dict(clip=cfg.clip, pa_noise_std=cfg.pa_noise_std, awgn_n0=cfg.awgn_n0, csi_eta=cfg.csi_eta,
               noise_key=inp["noise_key"], h_err=inp["h_err"])
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], device=DEV, max_batch=4,
               impair=imp)
    ch.step(torch.from_numpy(inp["s"]).to(DEV), torch.from_numpy(inp["idx"]).to(DEV))


def case_native():
    cfg = configs.C1
    inp = gen.make_inputs(cfg, list(range(4)))
    nat = fdpd.NativeChain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=4,
                           device=torch.device(DEV))
    c = torch.zeros(3, dtype=torch.int64).pin_memory()
    nat.run_host(torch.from_numpy(inp["s"]).pin_memory(), torch.from_numpy(inp["idx"]).pin_memory(), c)
    nat.run_host_qam(torch.from_numpy(inp["idx"]).pin_memory(), c)
    nat.close()


def case_c2():
    step_cfg(configs.C2, 2)


def case_cnn_tc():
    """C5-shaped tensor-core CNN (64-channel hidden layers) on 1 symbol x 2 UEs, both precisions;
    C3-shaped 32-channel stack."""
    rng = np.random.default_rng(1)
    for chans, Nd in (((2, 64, 64, 64, 64, 2), 3300), ((2, 32, 32, 32, 2), 1200)):
        n_par = sum(a * b * 9 + b for a, b in zip(chans[:-1], chans[1:]))
        params = torch.from_numpy((0.05 * rng.standard_normal(n_par)).astype(np.float32)).to(DEV)
        s = cr(rng, 1, 2, Nd, scale=0.7)
        for prec in (0, 1):
            fdpd.set_cnn_tc_precision(prec)
            fdpd.set_cnn_path(fdpd.CNN_TENSOR)
            fdpd.fdcnn_forward(params, chans, s)
        fdpd.set_cnn_tc_precision(0)
        fdpd.set_cnn_path(fdpd.CNN_AUTO)


def case_chain_cl():
    """N = 16384 cluster-split chain on 1 symbol x 2 antennas (C5 GMP shape), precoded input."""
    cfg = configs.C5
    rng = np.random.default_rng(2)
    inp = gen.make_inputs(cfg, [0])
    coef = torch.from_numpy(inp["coef"][:2]).to(DEV)
    X = cr(rng, 1, 2, cfg.N_d, scale=0.3)
    fdpd.chain_txrx_pre(X, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    fdpd.set_gmp_path(2)
    fdpd.chain_txrx_pre(X, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    fdpd.set_gmp_path(0)


def case_precode_tc():
    rng = np.random.default_rng(3)
    for (n, B, U, Nd) in ((2, 40, 32, 70), (3, 20, 12, 38)):
        P, s = cr(rng, B, U, Nd), cr(rng, n, U, Nd)
        for m in (fdpd.MATH_TF32, fdpd.MATH_FP32_TC):
            fdpd.precode(P, s, math=m)
            fdpd.precode_packed(fdpd.precode_pack(P), s, math=m)
        fdpd.precode(P, s)


def case_combine_tc():
    rng = np.random.default_rng(4)
    for (n, B, U, Nd) in ((2, 40, 32, 70), (33, 20, 12, 38)):
        XPA, h = cr(rng, n, B, Nd), cr(rng, U, B, Nd)
        idx = torch.from_numpy(rng.integers(0, 256, (n, U, Nd)).astype(np.uint16)).to(DEV)
        fdpd.set_combine_path(2)
        fdpd.ue_combine(XPA, h)
        fdpd.ue_combine_ser(XPA, h, 1.0, idx, 256)
        fdpd.set_combine_path(1)
        fdpd.ue_combine_ser(XPA, h, 1.0, idx, 256)
        fdpd.set_combine_path(0)


def case_zf():
    cfg = configs.C5
    inp = gen.make_inputs(cfg, [0])
    taps = torch.from_numpy(np.ascontiguousarray(inp["h_taps"][:, :, :64])).to(DEV)       # 64 antennas, k_zf (U = 32)
    fdpd.zf_precoder_build(taps, 256, 64, 0.3)


CASES = {"c1": case_c1, "c1_impair": case_c1_impair, "native": case_native, "c2": case_c2, "cnn_tc": case_cnn_tc,
         "chain_cl": case_chain_cl, "precode_tc": case_precode_tc, "combine_tc": case_combine_tc, "zf": case_zf}


def main():
    fdpd.lib()
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        torch.cuda.synchronize()
        print(f"case {nm}: ok", flush=True)


if __name__ == "__main__":
    main()

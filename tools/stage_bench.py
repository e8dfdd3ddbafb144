#!/usr/bin/env python
"""Times each stage of the hot path as its own C-ABI call (unfused) at a config's shape and
reports it against its own roofline (per-stage FLOP/s and the HBM fraction of
the bandwidth-bound stages, e.g. the standalone IDFT `ofdm_modulate`).

Inputs are resident on the device; L2 is flushed (256 MiB write) before every timed call;
CUDA events on the launching stream; median of the repetitions.
usage: python tools/stage_bench.py [CONFIG] [BATCH] [REPS]  -> one JSON line per stage"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402  (peaks, FLOP formulas)
from paper_2205_05158_b200 import fdpd  # noqa: E402
from workload import configs, gen  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    cfg = configs.get(name)
    n = int(sys.argv[2]) if len(sys.argv) > 2 else min(cfg.n_sym, 1024)
    reps = int(sys.argv[3]) if len(sys.argv) > 3 else 10
    pk = bench.peaks()
    alu_peak = 148 * 128 * 2 * pk["sm_max_mhz"] * 1e6 / 1e12       # TFLOP/s
    inp = gen.make_inputs(cfg, range(n))
    dev = "cuda"
    h_fd, P, alpha = fdpd.zf_precoder_build(torch.from_numpy(inp["h_taps"]).to(dev), cfg.N_ifft, cfg.N_d, cfg.rho)
    s = torch.from_numpy(inp["s"]).to(dev)
    idx = torch.from_numpy(inp["idx"].astype(np.int32)).to(dev).to(torch.uint16)
    coef = torch.from_numpy(inp["coef"]).to(dev)
    params = torch.from_numpy(inp["params"]).to(dev)
    B, U, N, Nd = cfg.B, cfg.U, cfg.N_ifft, cfg.N_d
    X = fdpd.precode(P, s)
    Ppk = fdpd.precode_pack(P) if U % 4 == 0 and U <= 32 else None
    x = fdpd.ofdm_modulate(X, N)
    y = fdpd.gmp_pa(x, coef, cfg.orders, cfg.L, cfg.M)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    st = torch.cuda.current_stream()

    def timed(fn):
        ts = []
        for i in range(reps + 2):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(st)
            fn()
            b.record(st)
            torch.cuda.synchronize()
            if i >= 2:
                ts.append(a.elapsed_time(b))
        return statistics.median(ts)

    c8 = 8  # bytes per complex64
    gmp_c = bench.gmp_flop_per_sample(cfg)
    stages = {
        # name: (callable, algorithmic bytes, algorithmic FLOPs)
        "fdcnn_forward": (lambda: fdpd.fdcnn_forward(params, cfg.chans, s), 2 * c8 * n * U * Nd,
                          2 * 9 * sum(a * b for a, b in zip(cfg.chans[:-1], cfg.chans[1:])) *
                          int(np.ceil(np.sqrt(Nd))) ** 2 * U * n),
        "precode": (lambda: fdpd.precode(P, s, out=X), c8 * (B * U * Nd + n * U * Nd + n * B * Nd), 8 * B * U * Nd * n),
        "precode_fp32tc": (lambda: fdpd.precode_packed(Ppk, s, out=X, math=fdpd.MATH_FP32_TC),
                           c8 * (B * U * Nd + n * U * Nd + n * B * Nd), 8 * B * U * Nd * n),
        "precode_tf32": (lambda: fdpd.precode_packed(Ppk, s, out=X, math=fdpd.MATH_TF32),
                         c8 * (B * U * Nd + n * U * Nd + n * B * Nd), 8 * B * U * Nd * n),
        "ofdm_modulate": (lambda: fdpd.ofdm_modulate(X, N, out=x), c8 * n * B * (Nd + N), 5 * N * np.log2(N) * B * n),
        "gmp_pa": (lambda: fdpd.gmp_pa(x, coef, cfg.orders, cfg.L, cfg.M, out=y), c8 * 2 * n * B * N, gmp_c * N * B * n),
        "ue_receive_ser": (lambda: fdpd.ue_receive_ser(y, h_fd, alpha, idx, cfg.M_qam),
                           c8 * (n * B * N + U * B * Nd + n * U * Nd) + 2 * n * U * Nd,
                           (5 * N * np.log2(N) + 8 * U * Nd) * B * n),
    }
    only = os.environ.get("STAGES")
    for k, (fn, nbytes, flops) in stages.items():
        if (only and k not in only.split(",")) or (Ppk is None and "tc" in k or Ppk is None and "tf32" in k):
            continue
        ms = timed(fn)
        gbs = nbytes / (ms * 1e-3) / 1e9
        tfs = flops / (ms * 1e-3) / 1e12
        print(json.dumps({"config": name, "batch": n, "stage": k, "ms": ms, "GBps": gbs, "hbm_frac": gbs / pk["hbm_gbs"],
                          "TFLOPs": tfs, "alu_frac": tfs / alu_peak, "bytes": int(nbytes), "flops": float(flops),
                          "hbm_peak_GBps": pk["hbm_gbs"], "alu_peak_TFLOPs": alu_peak}), flush=True)


if __name__ == "__main__":
    main()

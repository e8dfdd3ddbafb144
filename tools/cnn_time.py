#!/usr/bin/env python
"""Times fdcnn_forward on the SIMT and tensor-core paths (CUDA events, warm, L2 flushed).
usage: python tools/cnn_time.py [C2:1024 C3:256 ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from workload import configs  # noqa: E402


def flops(chans, U, N_d, n):
    S = int(np.ceil(np.sqrt(N_d)))
    return 2 * 9 * sum(a * b for a, b in zip(chans[:-1], chans[1:])) * S * S * U * n


def main():
    cases = sys.argv[1:] or ["C2:1024", "C3:256", "C4:256", "C5:64"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for case in cases:
        name, n = case.split(":")
        cfg = configs.get(name)
        n = int(n)
        g = torch.Generator(device="cuda").manual_seed(0)
        s = torch.randn((n, cfg.U, cfg.N_d), dtype=torch.complex64, device="cuda", generator=g) * 0.7
        n_par = sum(co * ci * 9 + co for ci, co in zip(cfg.chans[:-1], cfg.chans[1:]))
        params = torch.randn(n_par, device="cuda", generator=g) * 0.05
        out = {}
        paths = (("simt", fdpd.CNN_SIMT), ("tensor", fdpd.CNN_TENSOR))
        if os.environ.get("CNN_TIME_TENSOR_ONLY"):
            paths = paths[1:]
        for path, code in paths:
            fdpd.set_cnn_path(code)
            o = torch.empty_like(s)
            ws = None
            need = fdpd.lib().fdcnn_workspace_bytes(fdpd._ints(cfg.chans), len(cfg.chans) - 1, n, cfg.U, cfg.N_d)
            ws = fdpd._ws(need, s)
            for _ in range(2):
                fdpd.fdcnn_forward(params, cfg.chans, s, out=o, workspace=ws)
            ts = []
            for _ in range(5):
                flush.zero_()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fdpd.fdcnn_forward(params, cfg.chans, s, out=o, workspace=ws)
                e1.record()
                torch.cuda.synchronize()
                ts.append(e0.elapsed_time(e1))
            out[path] = (float(np.median(ts)), o.clone())
        fdpd.set_cnn_path(fdpd.CNN_AUTO)
        d = float("nan")
        if "simt" in out:
            d = (out["simt"][1] - out["tensor"][1]).abs().pow(2).sum().sqrt() / out["simt"][1].abs().pow(2).sum().sqrt()
        f = flops(cfg.chans, cfg.U, cfg.N_d, n)
        print(json.dumps({"config": name, "n_sym": n, "simt_ms": round(out["simt"][0], 4) if "simt" in out else None,
                          "tensor_ms": round(out["tensor"][0], 4),
                          "tensor_tflops": round(f / out["tensor"][0] / 1e9, 1),
                          "rel_simt_vs_tensor": float(d)}))


if __name__ == "__main__":
    main()

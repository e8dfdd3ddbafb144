#!/usr/bin/env python
"""Native runtime with the tensor-core GMP: run_device (twice), run_host and run_host_qam on the
same C5 batch; compares the SER counters and (run_device) y_hat bit for bit."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2205_05158_b200 import fdpd  # noqa: E402
from paper_2205_05158_b200.chain import Shapes  # noqa: E402
from workload import configs, gen  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
path = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = configs.get(name)
n = cfg.bench_batch
fdpd.set_gmp_path(path)
inp = gen.make_inputs(cfg, range(n))
nat = fdpd.NativeChain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=n)
s = torch.from_numpy(inp["s"]).cuda()
idx = torch.from_numpy(inp["idx"]).cuda()
res = []
for r in range(3):
    c = torch.zeros(3, dtype=torch.int64, device="cuda")
    yh = torch.empty_like(s)
    nat.run_device(s, idx, c, yhat=yh)
    torch.cuda.synchronize()
    res.append((c.cpu().tolist(), yh.clone()))
    print("run_device", r, res[-1][0], "yhat equal to first:", torch.equal(yh.view(torch.int64), res[0][1].view(torch.int64)),
          flush=True)
for r in range(2):
    ch = torch.zeros(3, dtype=torch.int64).pin_memory()
    nat.run_host(torch.from_numpy(inp["s"]).pin_memory(), torch.from_numpy(inp["idx"]).pin_memory(), ch)
    print("run_host", ch.tolist(), flush=True)
    cq = torch.zeros(3, dtype=torch.int64).pin_memory()
    nat.run_host_qam(torch.from_numpy(inp["idx"]).pin_memory(), cq)
    print("run_host_qam", cq.tolist(), flush=True)

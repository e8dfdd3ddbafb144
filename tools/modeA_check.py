#!/usr/bin/env python
"""Single-GPU validation of the Mode A (antenna-sharded) step on the CUDA path.

    python -m torch.distributed.run --nproc-per-node 2 --master-addr 127.0.0.1 --master-port P \
        tools/modeA_check.py C5 2 [fp32tc]

Both ranks run on cuda:0 with the gloo backend and host-staged collectives (NCCL refuses two
ranks on one device, and ranks whose kernels wait on each other must not share a GPU; here no
kernel waits on another rank — the collectives go through host copies).  Each rank runs
dist.AntennaShardedStep on its antenna half with chain.AntennaOps, then the single-GPU Mode S
step (all antennas) on its own symbols, and prints one JSON line: relative L2 of its y_hat
against the 1-rank run, and the world counters of both."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

from paper_2205_05158_b200 import dist as D  # noqa: E402
from paper_2205_05158_b200 import fdpd  # noqa: E402
from paper_2205_05158_b200.chain import AntennaOps, Chain, Shapes  # noqa: E402
from workload import configs, gen  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "C2"
    per = int(sys.argv[2]) if len(sys.argv) > 2 else 4
    math = sys.argv[3] if len(sys.argv) > 3 else ("fp32tc" if configs.get(name).U % 4 == 0 else "simt")
    dist.init_process_group("gloo")
    ws, rank = dist.get_world_size(), dist.get_rank()
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    fdpd.lib()
    cfg = configs.get(name)
    sh = Shapes.from_config(cfg)
    inp = gen.make_inputs(cfg, D.symbol_range(per, rank))
    b0, B_loc = D.antenna_shard(cfg.B, ws, rank)
    micro = 2 if per % 2 == 0 else 1
    ch = Chain(sh, inp["h_taps"], inp["coef"], inp["params"], device=dev, max_batch=ws * per // micro, b0=b0,
               B_loc=B_loc, precode_math=math)
    ops = AntennaOps(ch)
    peer = None
    if os.environ.get("MODEA_PEER") == "1":          # fused exchange: partial sums stored through CUDA IPC mappings
        assert ops.peer_ok(), "fused exchange needs 9 <= U <= 32"
        peer = D.PeerExchange(micro, per // micro, cfg.U, cfg.N_d, dev, host_staged=True)
    step = D.AntennaShardedStep(ops, per, cfg.U, cfg.N_d,
                                alloc=lambda shp: torch.empty(shp, dtype=torch.complex64, device=dev),
                                micro=micro, host_staged=True, peer=peer)
    s = torch.from_numpy(inp["s"]).to(dev)
    idx = torch.from_numpy(inp["idx"]).to(dev)
    counts = torch.zeros(3, dtype=torch.int64, device=dev)
    mine = torch.cat(step.step(s, idx, counts)).cpu().numpy()
    # the 1-rank reference: Mode S on this rank's symbols with every antenna
    ref = Chain(sh, inp["h_taps"], inp["coef"], inp["params"], device=dev, max_batch=per, precode_math=math)
    ref.split_precode = True
    c_ref = torch.zeros(3, dtype=torch.int64, device=dev)
    yhat_ref, _, _ = ref.step(s, idx, counts=c_ref)
    want = yhat_ref.cpu().numpy().astype(np.complex128)
    e = float(np.linalg.norm((mine - want).ravel()) / np.linalg.norm(want.ravel()))
    cr = c_ref.cpu()
    dist.all_reduce(cr)
    torch.cuda.synchronize()
    line = json.dumps({"rank": rank, "world": ws, "config": name, "per_rank": per, "micro": micro, "b0": b0,
                      "B_loc": B_loc, "precode": math, "peer": peer is not None, "yhat_rel_l2_vs_1rank": e, "counts_modeA": counts.cpu().tolist(),
                      "counts_1rank": cr.tolist()})
    out = os.environ.get("MODEA_OUT")
    if out:                              # one file per rank (the ranks' stdout interleave)
        with open(f"{out}.{rank}.json", "w") as f:
            f.write(line + "\n")
    print(line, flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()

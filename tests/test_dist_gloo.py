"""Multi-process (gloo, world_size 2, CPU) tests of the N>1 partitioning logic in
paper_2205_05158_b200/dist.py, with the fp64 oracle as the per-rank compute:
  * Mode S (symbol batches): per-rank SER counters all-reduced == unsharded counters.
  * Mode A (antennas): all-gathered symbol-sharded s_tilde == unsharded s_tilde, and
    the all-reduced per-rank partial channel sums == the unsharded received signal."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import fdpd_oracle as O
from workload import configs, gen


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


class OracleAntennaOps:
    """The per-rank compute of dist.AntennaShardedStep on the fp64 oracle (CPU test stand-in for
    chain.AntennaOps): this rank's antenna rows [b0, b0 + B_loc) of P, Hfd and the PA."""

    def __init__(self, cfg, inp, b0, B_loc):
        self.cfg, self.inp, self.b0, self.B_loc = cfg, inp, b0, B_loc
        self.Hfd = O.channel_fd(inp["h_taps"], cfg.N_ifft, cfg.N_d)
        self.P, self.alpha, _ = O.zf_precoder(self.Hfd, cfg.N_ifft, cfg.rho)

    def dpd(self, s, out):
        out.copy_(torch.from_numpy(O.fdcnn_forward(s.numpy(), self.inp["params"], self.cfg.chans, self.cfg.N_d)))

    def tx(self, st_all, XPA=None):
        cfg, sl = self.cfg, slice(self.b0, self.b0 + self.B_loc)
        X = O.precode(self.P[:, sl, :], st_all.numpy())
        return O.gmp_pa(O.ofdm_modulate(X, cfg.N_ifft), self.inp["coef"][sl], cfg.orders, cfg.L, cfg.M)

    def combine(self, y, out):
        out.copy_(torch.from_numpy(O.ue_receive(y, self.Hfd[:, :, self.b0:self.b0 + self.B_loc], self.cfg.N_d)))

    def slice(self, yhat, idx, counts):
        _, c = O.slice_ser(yhat.numpy(), self.alpha, idx.numpy(), self.cfg.M_qam)
        counts += torch.from_numpy(c)

    # fused exchange (dist.PeerExchange): what ue_combine_peer / ue_reduce_ser do, in numpy
    def combine_peer(self, y, peers, rank):
        from paper_2205_05158_b200 import dist as D
        part = O.ue_receive(y, self.Hfd[:, :, self.b0:self.b0 + self.B_loc], self.cfg.N_d)
        nm = peers[0].shape[1]
        for n in range(part.shape[0]):
            owner, slot, nl = D.peer_slot(n, nm, rank)
            peers[owner][slot, nl] = torch.from_numpy(part[n])

    def reduce_slice(self, recv, yhat, idx, counts):
        yhat.copy_(recv.sum(dim=0))
        self.slice(yhat, idx, counts)


def _worker(rank, world, port, mode, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2205_05158_b200 import dist as D
    try:
        cfg = configs.C1
        if mode in ("A_step", "A_step_peer"):
            per = 4
            syms = D.symbol_range(per, rank)
            inp_all = gen.make_inputs(cfg, range(per * world))
            inp = gen.make_inputs(cfg, syms)
            b0, B_loc = D.antenna_shard(cfg.B, world, rank)
            ops = OracleAntennaOps(cfg, inp_all, b0, B_loc)
            peer = None
            if mode == "A_step_peer":      # receive buffers in shared memory, mapped by the other rank
                mp.set_sharing_strategy("file_system")
                peer = D.PeerExchange(2, per // 2, cfg.U, cfg.N_d, "cpu", host_staged=True, dtype=torch.complex128)
            step = D.AntennaShardedStep(ops, per, cfg.U, cfg.N_d,
                                        alloc=lambda sh: torch.zeros(sh, dtype=torch.complex128), micro=2,
                                        host_staged=peer is not None, peer=peer)
            counts = torch.zeros(3, dtype=torch.int64)
            mine = step.step(torch.from_numpy(inp["s"].astype(np.complex128)), torch.from_numpy(inp["idx"]), counts)
            q.put((rank, (np.concatenate([m.numpy() for m in mine]), counts.numpy())))
        elif mode == "S":
            per = 3
            inp = gen.make_inputs(cfg, D.symbol_range(per, rank))
            out = O.run_config(cfg, inp)
            c = torch.tensor(out["counts"], dtype=torch.int64)
            D.allreduce_counts(c)
            q.put((rank, c.numpy()))
        else:
            n_total = 5
            inp = gen.make_inputs(cfg, range(n_total))
            s0, n_loc = D.split(n_total, world, rank)
            st_loc = O.fdcnn_forward(inp["s"][s0:s0 + n_loc], inp["params"], cfg.chans, cfg.N_d)
            st = D.allgather_symbols(torch.from_numpy(st_loc), n_total).numpy()
            Hfd = O.channel_fd(inp["h_taps"], cfg.N_ifft, cfg.N_d)
            P, alpha, _ = O.zf_precoder(Hfd, cfg.N_ifft, cfg.rho)
            b0, B_loc = D.antenna_shard(cfg.B, world, rank)
            X = O.precode(P[:, b0:b0 + B_loc, :], st)
            y = O.gmp_pa(O.ofdm_modulate(X, cfg.N_ifft), inp["coef"][b0:b0 + B_loc], cfg.orders, cfg.L, cfg.M)
            part = O.ue_receive(y, Hfd[:, :, b0:b0 + B_loc], cfg.N_d)
            yhat = D.allreduce_partial(torch.from_numpy(part)).numpy()
            q.put((rank, (st, yhat)))
    finally:
        dist.destroy_process_group()


def _run(mode, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, mode, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


def test_symbol_batch_counts_allreduce():
    res = _run("S")
    cfg = configs.C1
    want = O.run_config(cfg, gen.make_inputs(cfg, range(6)))["counts"]
    for r in (0, 1):
        assert np.array_equal(res[r], want)


def test_antenna_mode_allgather_and_partial_sum():
    res = _run("A")
    cfg = configs.C1
    full = O.run_config(cfg, gen.make_inputs(cfg, range(5)))
    for r in (0, 1):
        st, yhat = res[r]
        assert np.max(np.abs(st - full["s_tilde"])) < 1e-12
        assert np.max(np.abs(yhat - full["yhat"])) < 1e-12 * max(1.0, np.max(np.abs(full["yhat"])))


def test_antenna_sharded_step_matches_unsharded():
    """dist.AntennaShardedStep (Mode A, two micro-batches) over 2 gloo ranks: all_gather_into_tensor of
    s_tilde, local antennas, reduce_scatter_tensor of the partial received signals, counter all-reduce.
    Each rank's y_hat (its own symbols) and the world counters equal the unsharded oracle."""
    res = _run("A_step")
    cfg = configs.C1
    full = O.run_config(cfg, gen.make_inputs(cfg, range(8)))
    for r in (0, 1):
        yhat, counts = res[r]
        want = full["yhat"][4 * r:4 * r + 4]
        assert np.max(np.abs(yhat - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))
        assert np.array_equal(counts, full["counts"])


def test_antenna_sharded_step_fused_exchange():
    """The same step with dist.PeerExchange: each rank stores its partial received signals straight
    into the owner's receive buffer (mapped from the other process: shared memory here, CUDA IPC /
    NVLink peer memory on GPUs), one barrier, then the owner sums the slots in rank order."""
    res = _run("A_step_peer")
    cfg = configs.C1
    full = O.run_config(cfg, gen.make_inputs(cfg, range(8)))
    for r in (0, 1):
        yhat, counts = res[r]
        want = full["yhat"][4 * r:4 * r + 4]
        assert np.max(np.abs(yhat - want)) < 1e-12 * max(1.0, np.max(np.abs(want)))
        assert np.array_equal(counts, full["counts"])


def test_peer_slot_covers_every_buffer_once():
    from paper_2205_05158_b200 import dist as D
    for ws, nm in ((1, 3), (2, 2), (8, 4)):
        seen = set()
        for rank in range(ws):
            for n in range(ws * nm):
                owner, slot, nl = D.peer_slot(n, nm, rank)
                assert 0 <= owner < ws and slot == rank and 0 <= nl < nm
                seen.add((owner, slot, nl))
        assert len(seen) == ws * ws * nm


def test_split_covers_everything():
    from paper_2205_05158_b200 import dist as D
    for n in (1, 7, 64, 512):
        for w in (1, 2, 3, 8):
            parts = [D.split(n, w, r) for r in range(w)]
            assert sum(c for _, c in parts) == n
            assert all(parts[i][0] + parts[i][1] == parts[i + 1][0] for i in range(w - 1))

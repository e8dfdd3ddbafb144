"""Multi-core driver of the fp64 oracle, for bench.py's ``cpu_baseline`` leg and its
``--impl reference`` arm.

TEST / BENCH INFRASTRUCTURE ONLY (like fdpd_oracle itself): only ``bench.py``'s CPU legs
and ``tests/`` may import it; the product path never does.

It runs the functions of ``fdpd_oracle`` unchanged ("as it stands") on independent slices
of one OFDM symbol, spread over the host's cores with a fork-based process pool:

  * the FD-CNN per UE: with L_U = 1 (reading A2) every UE's S x S image goes
    through the network on its own, so ``fdcnn_forward`` on s[:, u:u+1] is the
    UE-u slice of the full call;
  * precode -> IDFT -> GMP -> receive per block of antennas: Eq. (1), Eq. (2)
     and the per-antenna PA of Eq. (7)/(9) act on each antenna
    row separately, and the received signal of Eq. (5) is a sum over antennas b,
    so ``ue_receive`` on a block of antennas returns that block's partial sum; the partial
    sums are added and ``slice_ser`` decides.

The ZF precoder (a2) is built once before timing, as on the GPU (reading A10).  No
arithmetic of the method lives here beyond adding the per-block partial sums of Eq. (5).
"""
from __future__ import annotations

import multiprocessing as mp
import os
import time

import numpy as np

from . import fdpd_oracle as O

_G: dict = {}        # per-run state; set in the parent before the pool forks (copy-on-write)


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def _limit_blas():
    try:
        from threadpoolctl import threadpool_limits
        return threadpool_limits(limits=1)
    except ImportError:  # pragma: no cover
        return None


def _cnn(args):
    i, u = args
    g = _G
    t0 = time.process_time()
    st = O.fdcnn_forward(g["s"][i:i + 1, u:u + 1], g["params"], g["cfg"].chans, g["cfg"].N_d)
    return u, st[0, 0], time.process_time() - t0


def _antennas(args):
    k, b0, b1 = args
    g, cfg = _G, _G["cfg"]
    t0 = time.process_time()
    X = O.precode(g["P"][:, b0:b1, :], g["st"][None])
    x = O.ofdm_modulate(X, cfg.N_ifft)
    y = O.gmp_pa(x, g["coef"][b0:b1], cfg.orders, cfg.L, cfg.M)
    g["parts"][k] = O.ue_receive(y, g["Hfd"][:, :, b0:b1], cfg.N_d)[0]
    return time.process_time() - t0


def _shared_complex(shape):
    """complex128 array in fork-shared memory (written by one process, read by the others)."""
    n = int(np.prod(shape))
    buf = mp.get_context("fork").RawArray("d", 2 * n)
    return np.frombuffer(buf, dtype=np.complex128, count=n).reshape(shape)


class OracleRunner:
    """The per-step stages of the hot path on the oracle, one OFDM
    symbol at a time over `workers` processes (1 = in-process, single core)."""

    def __init__(self, cfg, inp, workers=None):
        self.cfg = cfg
        self.workers = max(1, workers or host_cores())
        lim = None
        if self.workers == 1:
            lim = _limit_blas()
        Hfd = O.channel_fd(inp["h_taps"], cfg.N_ifft, cfg.N_d)
        P, alpha, _ = O.zf_precoder(Hfd, cfg.N_ifft, cfg.rho)
        _G.clear()
        nb = min(cfg.B, self.workers)
        self.blocks = [(cfg.B * k // nb, cfg.B * (k + 1) // nb) for k in range(nb)]
        _G.update(cfg=cfg, s=np.asarray(inp["s"]), idx=np.asarray(inp["idx"]), params=inp["params"],
                  coef=inp["coef"], P=P, Hfd=Hfd, alpha=alpha,
                  st=_shared_complex((cfg.U, cfg.N_d)), parts=_shared_complex((nb, cfg.U, cfg.N_d)))
        self.lim = lim
        self.pool = None
        if self.workers > 1:
            ctx = mp.get_context("fork")
            self.pool = ctx.Pool(self.workers, initializer=_limit_blas)

    def close(self):
        if self.pool is not None:
            self.pool.close()
            self.pool.join()
            self.pool = None
        if self.lim is not None:
            self.lim.restore_original_limits()
            self.lim = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def symbol(self, i):
        """Run symbol i (row of the inputs); returns (counts, wall s, summed task CPU s)."""
        cfg = self.cfg
        t0 = time.perf_counter()
        c0 = time.process_time()
        mp_map = self.pool.map if self.pool is not None else map
        st = _G["st"]
        cpu = 0.0
        for u, row, dt in mp_map(_cnn, [(i, u) for u in range(cfg.U)]):
            st[u] = row
            cpu += dt
        for dt in mp_map(_antennas, [(k, b0, b1) for k, (b0, b1) in enumerate(self.blocks)]):
            cpu += dt
        yhat = _G["parts"].sum(axis=0)
        _, counts = O.slice_ser(yhat[None], _G["alpha"], _G["idx"][i:i + 1], cfg.M_qam)
        wall = time.perf_counter() - t0
        if self.pool is not None:
            cpu += time.process_time() - c0      # the parent's share (partial sums, slicing)
        else:
            cpu = time.process_time() - c0
        return counts, wall, cpu

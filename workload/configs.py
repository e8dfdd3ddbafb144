"""The five BASELINE.json workload configurations, frozen.

This module holds only shapes and the synthetic-input recipe parameters
(no arithmetic of the method).  Sources:
  * BASELINE.json ``configs[0..4]`` (C1..C5).
  * SURVEY.md §8 config table and readings A6-A15.

N_ifft = os * N_fft everywhere (reading A8): the paper's N is the IDFT size
("oversampling rate R = N/N_d").
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Tuple


@dataclass(frozen=True)
class ChainConfig:
    name: str
    U: int                      # user equipments
    B: int                      # BS antennas
    N_fft: int                  # nominal FFT size (BASELINE)
    N_d: int                    # data subcarriers
    os: int                     # oversampling factor (BASELINE)
    M_qam: int                  # QAM order
    n_sym: int                  # OFDM symbols in one run
    T: int                      # channel taps
    pdp: str                    # "uniform" or "exp3dB" (BASELINE C2-C5)
    orders: Tuple[int, ...]     # GMP odd orders p (reading A13)
    L: int                      # GMP memory: l = 0..L (Eq. 9)
    M: int                      # GMP lag/lead cross-term length g = 1..M (paper's G)
    chans: Tuple[int, ...]      # FD-CNN channel list [2, hidden..., 2] (reading A1)
    spread: float               # per-antenna uniform relative coefficient spread (A15)
    seed: int
    rho: float = 0.3            # per-antenna TD RMS target (reading A12, BASELINE C1)
    w_std: float = 0.05         # CNN init std (reading A6, BASELINE C1)
    head: str = "residual"      # "residual": BASELINE conv stack (A1); "paper": conv + FC
    n_conv: int = 2             # paper head: N^Conv conv kernels
    # impairments; all off on the hot path (reading A11, A16)
    clip: float = 0.0           # PA saturation amplitude ("saturation point"), 0 = off
    pa_noise_std: float = 0.0   # PA measurement noise std per complex sample, CN(0, std^2)
    awgn_n0: float = 0.0        # AWGN variance N_0 at the UEs, per data subcarrier (unitary DFT)
    csi_eta: float = 0.0        # imperfect-CSI weight eta
    bench_batch: int = 0        # OFDM symbols per GPU per bench step (0: n_sym); SURVEY §8(d) streaming

    @property
    def N_ifft(self) -> int:
        return self.N_fft * self.os

    @property
    def S(self) -> int:
        """Side of the FD-CNN image: ceil(sqrt(N_d))."""
        return int(math.isqrt(self.N_d - 1)) + 1 if self.N_d > 0 else 0

    @property
    def Kp(self) -> int:
        return len(self.orders)

    @property
    def n_coef(self) -> int:
        """a: Kp(L+1); b and c: (Kp-1)(L+1)M each (SURVEY §8b flattening)."""
        return self.Kp * (self.L + 1) + 2 * (self.Kp - 1) * (self.L + 1) * self.M

    @property
    def n_layers(self) -> int:
        return len(self.chans) - 1

    @property
    def n_params(self) -> int:
        if self.head == "paper":
            return paper_head_n_params(self.n_conv, self.N_d)
        return sum(co * ci * 9 + co for ci, co in zip(self.chans[:-1], self.chans[1:]))


def paper_head_n_params(n_conv: int, N_d: int) -> int:
    """Paper FD-CNN: conv W1[n_conv][2][3][3] + b1[n_conv], FC W2[2 N_d][n_conv S^2] + b2[2 N_d]."""
    S = int(math.isqrt(N_d - 1)) + 1
    return n_conv * 2 * 9 + n_conv + 2 * N_d * n_conv * S * S + 2 * N_d


C1 = ChainConfig("C1", U=2, B=8, N_fft=64, N_d=36, os=2, M_qam=16, n_sym=4, T=4,
                 pdp="uniform", orders=(1, 3, 5), L=2, M=1, chans=(2, 4, 2),
                 spread=0.05, seed=0)
C2 = ChainConfig("C2", U=4, B=64, N_fft=1024, N_d=600, os=4, M_qam=64, n_sym=1024, T=8,
                 pdp="exp3dB", orders=(1, 3, 5, 7), L=4, M=2, chans=(2, 16, 16, 2),
                 spread=0.05, seed=1)
C3 = ChainConfig("C3", U=8, B=128, N_fft=2048, N_d=1200, os=4, M_qam=64, n_sym=2048, T=16,
                 pdp="exp3dB", orders=(1, 3, 5, 7), L=4, M=2, chans=(2, 32, 32, 32, 2),
                 spread=0.05, seed=2, bench_batch=512)
C4 = ChainConfig("C4", U=16, B=256, N_fft=4096, N_d=3300, os=4, M_qam=256, n_sym=2048, T=16,
                 pdp="exp3dB", orders=(1, 3, 5, 7, 9), L=6, M=3, chans=(2, 32, 32, 32, 2),
                 spread=0.05, seed=3, bench_batch=128)
C5 = ChainConfig("C5", U=32, B=512, N_fft=4096, N_d=3300, os=4, M_qam=256, n_sym=4096, T=16,
                 pdp="exp3dB", orders=(1, 3, 5, 7, 9), L=6, M=3,
                 chans=(2, 64, 64, 64, 64, 2), spread=0.10, seed=4, bench_batch=32)

# The paper's own workload with the paper's FD-CNN head (NEXT f2):
# N = 4096 IDFT, N_d = 384, U = 8, B = 32, 256-QAM, T = 10 uniform-PDP taps, FD-CNN
# ceil(sqrt(N_d)) = 20, L_U = 1, 3x3 kernels, stride 1, N^Conv = 2, ReLU, FC to 2 N_d.
# The PA keeps the odd-order GMP of reading A13 (K = 7 -> orders 1..7, memory 3, G = 1).
PAPER = ChainConfig("P", U=8, B=32, N_fft=1024, N_d=384, os=4, M_qam=256, n_sym=1024, T=10,
                    pdp="uniform", orders=(1, 3, 5, 7), L=3, M=1, chans=(2, 2), spread=0.05, seed=5,
                    head="paper", n_conv=2)

CONFIGS = {c.name: c for c in (C1, C2, C3, C4, C5, PAPER)}


def impaired(cfg: ChainConfig, clip: float = 1.0, pa_noise_std: float = None, awgn_n0: float = 1e-3,
             csi_eta: float = 1e-3) -> ChainConfig:
    """cfg with the paper's impairments switched on (NEXT f3).  In the normalised units of the
    chain (TD RMS rho = 0.3): clip at `clip`; PA noise std defaults to the paper's ratio
    0.053 V / 24.02 V of the saturation amplitude; eta = 0.001 as in P:204."""
    import dataclasses
    if pa_noise_std is None:
        pa_noise_std = clip * 0.053 / 24.02
    return dataclasses.replace(cfg, name=cfg.name + "i", clip=clip, pa_noise_std=pa_noise_std, awgn_n0=awgn_n0,
                               csi_eta=csi_eta)


def get(name: str) -> ChainConfig:
    return CONFIGS[name.upper()]

"""Seeded synthetic-input generator shared by the oracle tests and the CUDA path.

It holds NONE of the method's arithmetic (no CNN, ZF, precoding, DFT, GMP or
slicing).  It only draws the random inputs of the chain, with the recipe of
SURVEY.md §8(c) readings A6, A7, A10, A14, A15 and §8(d):

  stream 0  QAM indices, one substream per OFDM symbol n
  stream 1  Rayleigh taps H_t, T x U x B
  stream 2  per-antenna PA coefficient spread              (A15)
  stream 3  CNN weights, stream 4 CNN biases               (A6)

Every stream is ``numpy.random.Generator(PCG64(SeedSequence([seed, stream, index])))``
so any symbol can be regenerated alone (any rank, any subset).

The canonical arrays are float32 / complex64 (what the GPU consumes); the oracle
upcasts them exactly to float64 / complex128.

QAM symbol values (needed as the chain's input s) are the square M-QAM grid of
SPEC.md:116 / SURVEY §8(c) step 1: level 2i-(m-1), unit average energy.  The
oracle re-derives them independently from the indices (tests pin the two).
"""
from __future__ import annotations

import numpy as np

from .configs import ChainConfig

STREAM_SYMBOLS = 0
STREAM_CHANNEL = 1
STREAM_SPREAD = 2
STREAM_CNN_W = 3
STREAM_CNN_B = 4
STREAM_CSI = 5
STREAM_NOISE = 6


def rng(seed: int, stream: int, index: int = 0) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, stream, index])))


# ----------------------------------------------------------------------------- symbols
def qam_indices(cfg: ChainConfig, symbols) -> np.ndarray:
    """uint16 [len(symbols)][U][N_d], i.i.d. uniform in [0, M_qam)."""
    out = np.empty((len(symbols), cfg.U, cfg.N_d), dtype=np.uint16)
    for i, n in enumerate(symbols):
        out[i] = rng(cfg.seed, STREAM_SYMBOLS, int(n)).integers(
            0, cfg.M_qam, size=(cfg.U, cfg.N_d), dtype=np.uint16)
    return out


def qam_symbols(idx: np.ndarray, M_qam: int) -> np.ndarray:
    """complex64 points for indices: I = idx mod m, Q = idx div m (fixed map, A19)."""
    m = int(round(np.sqrt(M_qam)))
    scale = np.sqrt(3.0 / (2.0 * (M_qam - 1)))
    i = (idx.astype(np.int64) % m) * 2 - (m - 1)
    q = (idx.astype(np.int64) // m) * 2 - (m - 1)
    return ((i + 1j * q) * scale).astype(np.complex64)


# ----------------------------------------------------------------------------- channel
def pdp(cfg: ChainConfig) -> np.ndarray:
    """Power-delay profile p_t, sum 1: uniform 1/T or 3 dB/tap decay (BASELINE)."""
    if cfg.pdp == "uniform":
        p = np.full(cfg.T, 1.0 / cfg.T)
    elif cfg.pdp == "exp3dB":
        p = 10.0 ** (-0.3 * np.arange(cfg.T))
        p = p / p.sum()
    else:
        raise ValueError(cfg.pdp)
    return p


def channel_taps(cfg: ChainConfig) -> np.ndarray:
    """complex64 [T][U][B]; entries CN(0, p_t), i.i.d.."""
    g = rng(cfg.seed, STREAM_CHANNEL)
    z = g.standard_normal((cfg.T, cfg.U, cfg.B, 2))
    h = (z[..., 0] + 1j * z[..., 1]) * np.sqrt(pdp(cfg) / 2.0)[:, None, None]
    return h.astype(np.complex64)


def channel_taps_per_symbol(cfg: ChainConfig, symbols) -> np.ndarray:
    """complex64 [n][T][U][B]: one Rayleigh realisation per OFDM symbol (block-constant over one
    symbol; NEXT f4), substream index 1 + symbol (0 is the single-realisation channel)."""
    out = np.empty((len(symbols), cfg.T, cfg.U, cfg.B), dtype=np.complex64)
    sd = np.sqrt(pdp(cfg) / 2.0)[:, None, None]
    for i, n in enumerate(symbols):
        z = rng(cfg.seed, STREAM_CHANNEL, 1 + int(n)).standard_normal((cfg.T, cfg.U, cfg.B, 2))
        out[i] = (z[..., 0] + 1j * z[..., 1]) * sd
    return out


def csi_error_taps(cfg: ChainConfig) -> np.ndarray:
    """complex64 [T][U][B] H^err ~ CN(0, I) per tap entry."""
    g = rng(cfg.seed, STREAM_CSI)
    z = g.standard_normal((cfg.T, cfg.U, cfg.B, 2))
    return ((z[..., 0] + 1j * z[..., 1]) / np.sqrt(2.0)).astype(np.complex64)


def noise_key(cfg: ChainConfig) -> int:
    """64-bit key of the counter-based (Philox4x32-10) noise generator shared by the oracle
    and the GPU; counters are global sample indices, so any shard regenerates its noise."""
    return int(np.random.SeedSequence([cfg.seed, STREAM_NOISE]).generate_state(1, dtype=np.uint64)[0])


# ----------------------------------------------------------------------------- PA bank
# Nominal a_{p,0} (BASELINE C1 gives p = 1, 3, 5; 7 and 9 invented, reading A14).
NOMINAL_A0 = {1: 1.0 + 0.0j, 3: -0.08 + 0.02j, 5: 0.01 - 0.005j,
              7: -1e-3 + 5e-4j, 9: 1e-4 - 5e-5j}


def gmp_nominal(cfg: ChainConfig) -> np.ndarray:
    """complex128 [n_coef] in the flattened order of SURVEY §8(b):
    a[p][l] for p in orders, l = 0..L; then b[p][l][g] for p >= 3, l, g = 1..M;
    then c[p][l][g] likewise.  Values per reading A14."""
    a = []
    for p in cfg.orders:
        for l in range(cfg.L + 1):
            a.append(NOMINAL_A0[p] * (1.0 if l == 0 else 0.05 * 0.5 ** (l - 1)))
    bc = []
    for p in cfg.orders[1:]:
        for l in range(cfg.L + 1):
            for g in range(1, cfg.M + 1):
                bc.append(NOMINAL_A0[p] * 0.02 * 0.5 ** l * 0.5 ** (g - 1))
    return np.array(a + bc + bc, dtype=np.complex128)


def gmp_coefficients(cfg: ChainConfig) -> np.ndarray:
    """complex64 [B][n_coef]: nominal * (1 + delta), delta ~ U[-spread, spread] real,
    i.i.d. per (antenna, coefficient), frozen per seed (reading A15)."""
    nom = gmp_nominal(cfg)
    d = rng(cfg.seed, STREAM_SPREAD).uniform(-cfg.spread, cfg.spread, size=(cfg.B, nom.size))
    return (nom[None, :] * (1.0 + d)).astype(np.complex64)


def gmp_identity(cfg: ChainConfig) -> np.ndarray:
    """a_{1,0} = 1, all else 0 on every antenna: the linear PA of PAPER.md:94."""
    c = np.zeros((cfg.B, cfg.n_coef), dtype=np.complex64)
    c[:, 0] = 1.0
    return c


# ----------------------------------------------------------------------------- CNN
def cnn_params(cfg: ChainConfig) -> np.ndarray:
    """float32 flat parameter vector: per layer W[co][ci][3][3] then b[co].
    All entries N(0, w_std^2) (reading A6)."""
    gw = rng(cfg.seed, STREAM_CNN_W)
    gb = rng(cfg.seed, STREAM_CNN_B)
    parts = []
    for ci, co in zip(cfg.chans[:-1], cfg.chans[1:]):
        parts.append(gw.normal(0.0, cfg.w_std, size=co * ci * 9))
        parts.append(gb.normal(0.0, cfg.w_std, size=co))
    return np.concatenate(parts).astype(np.float32)


def cnn_zero(cfg: ChainConfig) -> np.ndarray:
    return np.zeros(cfg.n_params, dtype=np.float32)


def paper_head_params(cfg: ChainConfig) -> np.ndarray:
    """Paper FD-CNN head, random init: conv N(0, 0.05^2), FC N(0, 1/fan_in).
    Layout: W1[n_conv][2][3][3], b1[n_conv], W2[2 N_d][n_conv S^2], b2[2 N_d]."""
    gw = rng(cfg.seed, STREAM_CNN_W)
    gb = rng(cfg.seed, STREAM_CNN_B)
    K = cfg.n_conv * cfg.S * cfg.S
    parts = [gw.normal(0.0, cfg.w_std, size=cfg.n_conv * 18), gb.normal(0.0, cfg.w_std, size=cfg.n_conv),
             gw.normal(0.0, 1.0 / np.sqrt(K), size=2 * cfg.N_d * K), gb.normal(0.0, cfg.w_std, size=2 * cfg.N_d)]
    return np.concatenate(parts).astype(np.float32)


def paper_head_identity(cfg: ChainConfig, offset: float = 4.0) -> np.ndarray:
    """A paper head that passes s through: conv kernel 0 = Re, kernel 1 = Im (centre tap) with
    bias +offset so ReLU never clips (|s| < offset), FC selects pixel i of each map, bias -offset.
    Only kernels 0 and 1 are used (n_conv >= 2)."""
    S, Nd, n_conv = cfg.S, cfg.N_d, cfg.n_conv
    W1 = np.zeros((n_conv, 2, 3, 3))
    W1[0, 0, 1, 1] = 1.0
    W1[1, 1, 1, 1] = 1.0
    b1 = np.zeros(n_conv)
    b1[:2] = offset
    W2 = np.zeros((2 * Nd, n_conv * S * S))
    for i in range(Nd):
        W2[i, 0 * S * S + i] = 1.0
        W2[Nd + i, 1 * S * S + i] = 1.0
    b2 = np.full(2 * Nd, -offset)
    return np.concatenate([W1.ravel(), b1, W2.ravel(), b2]).astype(np.float32)


# ----------------------------------------------------------------------------- bundle
def make_inputs(cfg: ChainConfig, symbols=None, *, zero_cnn=False, linear_pa=False):
    """All inputs of one run (or of a subset of its symbols)."""
    if symbols is None:
        symbols = range(cfg.n_sym)
    symbols = list(symbols)
    idx = qam_indices(cfg, symbols)
    return {
        "symbols": np.array(symbols, dtype=np.int64),
        "idx": idx,
        "s": qam_symbols(idx, cfg.M_qam),
        "h_taps": channel_taps(cfg),
        "h_err": csi_error_taps(cfg),
        "noise_key": noise_key(cfg),
        "coef": gmp_identity(cfg) if linear_pa else gmp_coefficients(cfg),
        "params": (paper_head_identity(cfg) if zero_cnn else paper_head_params(cfg)) if cfg.head == "paper"
        else (cnn_zero(cfg) if zero_cnn else cnn_params(cfg)),
    }

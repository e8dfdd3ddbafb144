"""Pins for the impairment stages of the oracle (NEXT f3: PA clip + measurement noise P:202,
AWGN P:65, imperfect CSI P:85) and their counter-based RNG."""
import dataclasses
import math

import numpy as np

from oracle import fdpd_oracle as O
from workload import configs, gen

# Known-answer vectors of Philox4x32-10 (Salmon, Moraes, Dror, Shaw, "Parallel random numbers:
# as easy as 1, 2, 3", SC'11; the Random123 distribution's kat_vectors): (counter, key) -> output.
KAT = [((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
       ((0xFFFFFFFF,) * 4, (0xFFFFFFFF, 0xFFFFFFFF), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
       ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
        (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1))]


def test_philox_known_answers():
    for ctr, key, want in KAT:
        got = O.philox4x32_10(np.array(ctr, dtype=np.uint64), key)
        assert tuple(int(v) for v in got) == want


def test_gaussian_moments_and_independence():
    x = O.complex_gaussian(np.arange(400_000), O.STREAM_AWGN, 12345, 2.0)
    assert abs(np.mean(x)) < 0.01
    assert abs(np.mean(np.abs(x) ** 2) / 4.0 - 1) < 0.01            # E|x|^2 = std^2
    assert abs(np.mean(x.real ** 2) / 2.0 - 1) < 0.01               # circular: half per axis
    assert abs(np.mean(x.real * x.imag)) < 0.01
    y = O.complex_gaussian(np.arange(400_000), O.STREAM_PA_NOISE, 12345, 2.0)
    assert abs(np.mean(x * np.conj(y))) < 0.02                       # streams independent
    assert np.array_equal(O.complex_gaussian(np.arange(10, 20), 2, 7, 1.0),
                          O.complex_gaussian(np.arange(30)[10:20], 2, 7, 1.0))


def test_clip_keeps_phase_and_bounds_magnitude():
    rng = np.random.default_rng(0)
    y = (rng.standard_normal((2, 3, 64)) + 1j * rng.standard_normal((2, 3, 64)))
    c = O.pa_impair(y, 1.0, 0.0, 0, [0, 1], 3)
    assert np.max(np.abs(c)) <= 1.0 + 1e-12
    big = np.abs(y) > 1.0
    assert np.allclose(np.angle(c[big]), np.angle(y[big]))
    assert np.array_equal(c[~big], y[~big])


def test_csi_estimate_statistics():
    cfg = dataclasses.replace(configs.C5, csi_eta=0.001)
    h, e = gen.channel_taps(cfg), gen.csi_error_taps(cfg)
    he = O.csi_estimate(h, e, 0.25)
    d = he - np.sqrt(0.75) * h
    assert abs(np.var(d) / 0.25 - 1) < 0.02                          # var(H_est - sqrt(1-eta) H) = eta


def _qfunc(x):
    return 0.5 * math.erfc(x / math.sqrt(2.0))


def test_awgn_qpsk_ser_closed_form():
    """B = U = 1, T = 1 flat channel, linear PA, no DPD, QPSK: SER = 2Q(sqrt(SNR)) - Q^2
    with SNR = alpha^2 / N_0 (E|s|^2 = 1, genie alpha)."""
    base = configs.ChainConfig("awgn", U=1, B=1, N_fft=64, N_d=64, os=2, M_qam=4, n_sym=3000, T=1,
                               pdp="uniform", orders=(1,), L=0, M=0, chans=(2, 2), spread=0.0, seed=21)
    inp = gen.make_inputs(base, zero_cnn=True, linear_pa=True)
    alpha = O.zf_precoder(O.channel_fd(inp["h_taps"], base.N_ifft, base.N_d), base.N_ifft, base.rho)[1]
    snr = 2.576 ** 2                                                 # per-axis error ~ 5e-3
    cfg = dataclasses.replace(base, awgn_n0=alpha ** 2 / snr)
    out = O.run_config(cfg, inp)
    p = _qfunc(math.sqrt(snr))
    want = 2 * p - p * p
    ser = out["counts"][0] / out["counts"][1]
    assert abs(ser / want - 1) < 0.10


def test_redraw_with_repeated_taps_equals_single_realisation():
    """NEXT f4 oracle: per-symbol channels that all equal the run's channel reproduce run_config."""
    cfg = configs.C1
    inp = gen.make_inputs(cfg)
    taps = np.repeat(inp["h_taps"][None], cfg.n_sym, axis=0)
    a = O.run_config_redraw(cfg, inp, taps)
    b = O.run_config(cfg, inp)
    assert np.allclose(a["yhat"], b["yhat"], rtol=0, atol=1e-13) and np.array_equal(a["counts"], b["counts"])
    assert np.allclose(a["alpha"], b["alpha"])


def test_redraw_channels_differ_per_symbol():
    cfg = configs.C2
    t = gen.channel_taps_per_symbol(cfg, [0, 1, 0])
    assert np.array_equal(t[0], t[2]) and not np.allclose(t[0], t[1])
    p = np.mean(np.abs(gen.channel_taps_per_symbol(cfg, range(64)).astype(np.complex128)) ** 2, axis=(0, 2, 3))
    assert abs(p.sum() - 1) < 0.03                       # PDP normalised per realisation on average

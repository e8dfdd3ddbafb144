"""Generator determinism and recipe statistics."""
import numpy as np

from workload import configs, gen


def test_determinism_and_substreams():
    cfg = configs.C2
    a = gen.make_inputs(cfg, range(6))
    b = gen.make_inputs(cfg, range(6))
    for k in a:
        assert np.array_equal(a[k], b[k])
    sub = gen.make_inputs(cfg, [4, 2])          # any subset regenerates identically
    assert np.array_equal(sub["idx"][0], a["idx"][4]) and np.array_equal(sub["idx"][1], a["idx"][2])


def test_config_derived_sizes():
    base = [configs.C1, configs.C2, configs.C3, configs.C4, configs.C5]
    assert [c.N_ifft for c in base] == [128, 4096, 8192, 16384, 16384]
    assert [c.S for c in base] == [6, 25, 35, 58, 58]
    assert [c.n_coef for c in base] == [21, 80, 80, 203, 203]
    assert [c.n_params for c in base] == [150, 2914, 19682, 19682, 113154]
    p = configs.PAPER                       # paper workload P:204-206 with the paper head
    assert (p.N_ifft, p.S, p.n_params) == (4096, 20, 2 * 19 + 768 * 800 + 768)


def test_channel_pdp_and_moments():
    cfg = configs.C5
    h = gen.channel_taps(cfg).astype(np.complex128)
    p = np.mean(np.abs(h) ** 2, axis=(1, 2))
    assert abs(p.sum() - 1.0) < 0.01
    assert abs(p[1] / p[0] - 10 ** -0.3) < 0.05
    assert abs(np.mean(h)) < 0.01


def test_spread_statistics():
    cfg = configs.C5
    nom = gen.gmp_nominal(cfg)
    c = gen.gmp_coefficients(cfg).astype(np.complex128)
    d = (c / nom[None, :]).real - 1.0
    assert np.max(np.abs(d)) <= cfg.spread + 1e-6
    assert abs(np.std(d) - cfg.spread / np.sqrt(3.0)) < 0.003


def test_qam_indices_uniform():
    cfg = configs.C4
    idx = gen.qam_indices(cfg, range(4))
    assert idx.min() == 0 and idx.max() == cfg.M_qam - 1
    assert abs(idx.mean() - (cfg.M_qam - 1) / 2) < 1.0

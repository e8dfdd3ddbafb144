"""GPU parity of the impairment stages (NEXT f3: PA clip + measurement noise P:202, AWGN P:65,
imperfect CSI P:85) against the fp64 oracle: the noise comes from the same Philox4x32-10
counters on both sides, so waveforms, received signals and decisions are compared directly."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fdpd_oracle as O
from workload import configs, gen

pytestmark = pytest.mark.gpu
TOL = 2e-5


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2205_05158_b200 import fdpd
    fdpd.lib()
    return fdpd


def rel(a, b):
    a, b = np.asarray(a, np.complex128), np.asarray(b, np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / np.linalg.norm(b.ravel()))


def _impair_dict(cfg, inp):
    return dict(clip=cfg.clip, pa_noise_std=cfg.pa_noise_std, awgn_n0=cfg.awgn_n0, csi_eta=cfg.csi_eta,
                noise_key=inp["noise_key"], h_err=inp["h_err"])


def _near(yhat, alpha, M):
    m = int(round(np.sqrt(M)))
    c = 1.0 / np.sqrt(2.0 * (M - 1) / 3.0)
    z = np.asarray(yhat, np.complex128) / alpha
    near = np.zeros(z.shape, bool)
    for v in (z.real / c, z.imag / c):
        bnd = 2.0 * np.round(v / 2.0)
        near |= (np.abs(v - bnd) < 1e-4 / c) & (np.abs(bnd) <= m - 2)
    return near


@pytest.mark.parametrize("name,clip", [("C1", 0.5), ("C2", 0.6), ("P", 0.6)])
def test_impaired_chain_vs_oracle(F, name, clip):
    from paper_2205_05158_b200.chain import Chain, Shapes
    cfg = configs.impaired(configs.get(name), clip=clip)
    nsym = 4 if name == "C1" else 3
    sym0 = 0 if name == "C1" else 100
    # the random-init paper head shrinks the signal far below any clip: use its identity head there
    inp = gen.make_inputs(cfg, range(sym0, sym0 + nsym), zero_cnn=(cfg.head == "paper"))
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=nsym,
               impair=_impair_dict(cfg, inp))
    s = torch.from_numpy(inp["s"]).cuda()
    idx = torch.from_numpy(inp["idx"]).cuda()
    dec = torch.zeros(idx.shape, dtype=torch.uint16, device="cuda")
    yhat, counts, _ = ch.step(s, idx, dec=dec, sym0=sym0)
    torch.cuda.synchronize()
    o = O.run_config(cfg, inp)
    assert abs(ch.alpha / o["alpha"] - 1) < 1e-6
    assert rel(ch.y[:nsym].cpu().numpy(), o["y"]) < TOL
    assert rel(yhat.cpu().numpy(), o["yhat"]) < TOL
    clipped = np.mean(np.abs(O.gmp_pa(o["x"], inp["coef"], cfg.orders, cfg.L, cfg.M)) > clip)
    assert clipped > 1e-4                                            # the clip is exercised
    near = _near(o["yhat"], o["alpha"], cfg.M_qam)
    assert np.array_equal(dec.cpu().numpy()[~near], o["dec"][~near])
    c = counts.cpu().numpy()
    assert abs(int(c[0]) - int(o["counts"][0])) <= int(near.sum())


def test_noise_is_batch_invariant(F):
    """Noise indices are global: two half batches with sym0 offsets == one batch."""
    from paper_2205_05158_b200.chain import Chain, Shapes
    cfg = configs.impaired(configs.C1, clip=0.5)
    inp = gen.make_inputs(cfg)
    sh = Shapes.from_config(cfg)
    ch = Chain(sh, inp["h_taps"], inp["coef"], inp["params"], max_batch=4, impair=_impair_dict(cfg, inp))
    s = torch.from_numpy(inp["s"]).cuda()
    idx = torch.from_numpy(inp["idx"]).cuda()
    full, _, _ = ch.step(s, idx)
    full = full.clone()
    a, _, _ = ch.step(s[:2], idx[:2], sym0=0)
    a = a.clone()
    b, _, _ = ch.step(s[2:], idx[2:], sym0=2)
    assert torch.equal(torch.cat([a, b]), full)


def test_pa_noise_statistics(F):
    """Linear PA, no clip: y - y_clean is the measurement noise, CN(0, std^2)."""
    cfg = configs.C2
    inp = gen.make_inputs(cfg, range(8), linear_pa=True)
    h_fd, P, alpha = F.zf_precoder_build(torch.from_numpy(inp["h_taps"]).cuda(), cfg.N_ifft, cfg.N_d, cfg.rho)
    s = torch.from_numpy(inp["s"]).cuda()
    coef = torch.from_numpy(inp["coef"]).cuda()
    y0, _ = F.chain_txrx(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    imp = F.make_impairments(pa_noise_std=0.01, noise_key=inp["noise_key"])
    y1, _ = F.chain_txrx_ex(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft, imp)
    d = (y1 - y0).cpu().numpy().astype(np.complex128)
    assert abs(np.mean(np.abs(d) ** 2) / 1e-4 - 1) < 0.01
    assert abs(np.mean(d)) < 1e-4

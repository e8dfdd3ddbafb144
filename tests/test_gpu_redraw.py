"""GPU parity of the per-symbol channel redraw path (NEXT f4): batched ZF build on the hot
path, per-symbol precoders / channels / alpha, against the per-symbol fp64 oracle."""
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


@pytest.mark.parametrize("name,nsym,impair", [("C1", 4, False), ("C2", 3, False), ("C1", 4, True), ("P", 2, False)])
def test_redraw_chain_vs_oracle(F, name, nsym, impair):
    from paper_2205_05158_b200.chain import Chain, Shapes
    cfg = configs.get(name)
    if impair:
        cfg = configs.impaired(cfg, clip=0.5, csi_eta=0.0)
    syms = list(range(nsym))
    inp = gen.make_inputs(cfg, syms)
    taps = gen.channel_taps_per_symbol(cfg, syms)
    imp = dict(clip=cfg.clip, pa_noise_std=cfg.pa_noise_std, awgn_n0=cfg.awgn_n0, noise_key=inp["noise_key"]) \
        if impair else None
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=nsym, impair=imp)
    s = torch.from_numpy(inp["s"]).cuda()
    idx = torch.from_numpy(inp["idx"]).cuda()
    dec = torch.zeros(idx.shape, dtype=torch.uint16, device="cuda")
    yhat, counts, _ = ch.step_redraw(s, idx, torch.from_numpy(taps).cuda(), dec=dec)
    torch.cuda.synchronize()
    o = O.run_config_redraw(cfg, inp, taps)
    assert int(ch.zf_status.item()) == 0
    assert np.max(np.abs(ch.alpha_all.cpu().numpy() / o["alpha"] - 1)) < 1e-6
    assert rel(ch.P_all.cpu().numpy(), o["P"].transpose(0, 2, 3, 1)) < TOL
    assert rel(ch.y[:nsym].cpu().numpy(), o["y"]) < TOL
    assert rel(yhat.cpu().numpy(), o["yhat"]) < TOL
    c = counts.cpu().numpy()
    assert c[1] == o["counts"][1] and abs(int(c[0]) - int(o["counts"][0])) <= int(o["counts"][2]) + int(c[2])


def test_redraw_invariant(F):
    """Zero CNN + linear PA + noiseless per-symbol ZF: z = s, SER = 0, with per-symbol alpha."""
    from paper_2205_05158_b200.chain import Chain, Shapes
    cfg = configs.C2
    inp = gen.make_inputs(cfg, range(8), zero_cnn=True, linear_pa=True)
    taps = gen.channel_taps_per_symbol(cfg, range(8))
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=8)
    yhat, counts, _ = ch.step_redraw(torch.from_numpy(inp["s"]).cuda(), torch.from_numpy(inp["idx"]).cuda(),
                                     torch.from_numpy(taps).cuda())
    z = yhat.cpu().numpy() / ch.alpha_all.cpu().numpy()[:, None, None]
    assert rel(z, inp["s"]) < TOL and int(counts[0]) == 0

"""Pins for the fp64 oracle (CPU only): each oracle function is checked against
something other than itself — closed forms, hand-computed fixtures (tests/golden),
library special cases, brute force on tiny inputs, and invariants of the paper.
See DESIGN.md "Parity pins" for the table."""
import os

import numpy as np
import pytest

from oracle import fdpd_oracle as O
from workload import configs, gen

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _read_golden(name):
    rows = {}
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if not line or line.startswith("#"):
                continue
            kind, i, re, im = line.split()
            rows.setdefault(kind, {})[int(i)] = float(re) + 1j * float(im)
    return {k: np.array([v[i] for i in sorted(v)]) for k, v in rows.items()}


def _crandn(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


# ============================================================================ QAM
@pytest.mark.parametrize("M", [4, 16, 64, 256])
def test_qam_unit_energy_closed_form(M):
    pts = O.qam_points(np.arange(M), M)
    assert len(np.unique(np.round(pts, 12))) == M
    assert abs(np.mean(np.abs(pts) ** 2) - 1.0) < 1e-14      # E|s|^2 = 1 exactly


def test_qpsk_points():
    pts = O.qam_points(np.arange(4), 4)
    want = {(1 + 1j) / np.sqrt(2), (1 - 1j) / np.sqrt(2), (-1 + 1j) / np.sqrt(2), (-1 - 1j) / np.sqrt(2)}
    for p in pts:
        assert min(abs(p - w) for w in want) < 1e-15


@pytest.mark.parametrize("M", [16, 64, 256])
def test_generator_symbols_match_oracle_points(M):
    idx = np.arange(M, dtype=np.uint16)
    assert np.array_equal(gen.qam_symbols(idx, M), O.qam_points(idx, M).astype(np.complex64))


@pytest.mark.parametrize("M", [4, 16, 64, 256])
def test_slicer_exact_and_perturbed_points(M):
    idx = np.arange(M)
    pts = O.qam_points(idx, M)
    alpha = 0.7
    dec, cnt = O.slice_ser(alpha * pts[None, None, :], alpha, idx[None, None, :], M)
    assert np.array_equal(dec[0, 0], idx) and cnt[0] == 0 and cnt[2] == 0
    dmin = 2.0 / np.sqrt(2.0 * (M - 1) / 3.0)
    rng = np.random.default_rng(5)
    for _ in range(4):
        ang = rng.uniform(0, 2 * np.pi, M)
        off = 0.49 * dmin * np.maximum(abs(np.cos(ang)), abs(np.sin(ang))) ** -1 * np.exp(1j * ang) * 0.7
        dec, cnt = O.slice_ser(alpha * (pts + off)[None, None, :], alpha, idx[None, None, :], M)
        assert cnt[0] == 0


def test_slicer_errors_ties_and_near_boundary():
    M = 16
    c = 1.0 / np.sqrt(10.0)
    # level units: v = 2.0 is the boundary between levels 1 and 3 -> ties go up (A18)
    z = np.array([2.0 * c + 0j, 1.99 * c + 0j, 5.0 * c + 0j, -7.5 * c + 0j])
    # levels -3,-1,1,3 have I-index 0..3: v=2 (tie) -> 3 -> 3; 1.99 -> 1 -> 2; 5 -> clip 3 -> 3;
    # -7.5 -> 2*floor(-3.75)+1 = -7 -> clip -3 -> 0
    dec, cnt = O.slice_ser(z[None, None, :], 1.0, np.zeros((1, 1, 4), np.int64), M)
    lvl_i = dec[0, 0] % 4
    assert list(lvl_i) == [3, 2, 3, 0]
    # Q axis: imag 0 -> v = 0 is an interior boundary (between -1 and 1): near for all four
    assert cnt[2] == 4
    z2 = np.array([1.0 * c + 1j * c])
    _, cnt2 = O.slice_ser(z2[None, None, :], 1.0, np.array([[[2 + 4 * 2]]]), M)
    assert cnt2[0] == 0 and cnt2[2] == 0
    # a boundary just outside eps is not near; inside is near
    eps = 1e-4
    z3 = np.array([(2.0 + 1.5 * eps / c) * c + 1j * c, (2.0 + 0.5 * eps / c) * c + 1j * c])
    _, cnt3 = O.slice_ser(z3[None, None, :], 1.0, np.array([[[3 + 8, 3 + 8]]]), M, eps=eps)
    assert cnt3[2] == 1 and cnt3[0] == 0


# ============================================================================ IDFT / DFT
def _brute_idft(Xfull):
    N = Xfull.shape[-1]
    n = np.arange(N)
    W = np.exp(2j * np.pi * np.outer(n, n) / N) / np.sqrt(N)
    return Xfull @ W.T


@pytest.mark.parametrize("N,Nd", [(128, 36), (256, 100), (64, 64)])
def test_ofdm_modulate_vs_brute_force(N, Nd):
    rng = np.random.default_rng(1)
    X = _crandn(rng, 2, 3, Nd)
    full = np.zeros((2, 3, N), complex)
    for j in range(Nd):                                   # bins written out by hand (A7)
        k = j - Nd // 2 if j >= Nd // 2 else N - (Nd // 2 - j)
        full[..., k] = X[..., j]
    assert np.max(np.abs(O.ofdm_modulate(X, N) - _brute_idft(full))) < 1e-12


def test_idft_impulse_and_tone():
    N, Nd = 4, 4
    # DC data subcarrier is j = Nd/2 (A7); e_0 -> 1/2 [1,1,1,1]
    X = np.zeros((1, 1, Nd), complex)
    X[0, 0, Nd // 2] = 1
    assert np.allclose(O.ofdm_modulate(X, N)[0, 0], 0.5 * np.ones(4), atol=1e-15)
    # bin 1 is j = Nd/2 + 1 -> 1/2 [1, j, -1, -j]
    X = np.zeros((1, 1, Nd), complex)
    X[0, 0, Nd // 2 + 1] = 1
    assert np.allclose(O.ofdm_modulate(X, N)[0, 0], 0.5 * np.array([1, 1j, -1, -1j]), atol=1e-15)
    # single tone: constant magnitude
    X = np.zeros((1, 1, 36), complex)
    X[0, 0, 7] = 2 - 1j
    x = O.ofdm_modulate(X, 128)
    assert np.allclose(np.abs(x), np.abs(2 - 1j) / np.sqrt(128), atol=1e-14)


def test_parseval_and_round_trip():
    rng = np.random.default_rng(2)
    X = _crandn(rng, 3, 5, 600)
    x = O.ofdm_modulate(X, 4096)
    assert abs(np.sum(np.abs(x) ** 2) - np.sum(np.abs(X) ** 2)) < 1e-9 * np.sum(np.abs(X) ** 2)
    # the receive DFT with an identity channel (U = B) returns X (Eq. 2 then Eq. 4)
    H = np.broadcast_to(np.eye(5), (600, 5, 5))
    assert np.max(np.abs(O.ue_receive(x, H, 600) - X)) < 1e-12


# ============================================================================ FD-CNN
def test_fdcnn_golden_hand_computed():
    g = _read_golden("fdcnn_2x2.txt")
    W = np.zeros((2, 2, 3, 3))
    W[0, 0] = 1.0
    W[1, 1, 0, 0] = 1.0
    params = np.concatenate([W.ravel(), [0.5, -0.25]])
    st = O.fdcnn_forward(g["s"][None, None, :], params, (2, 2), 3)
    assert np.max(np.abs(st[0, 0] - g["st"])) < 1e-14


def test_fdcnn_zero_weights_is_identity():
    cfg = configs.C2
    inp = gen.make_inputs(cfg, range(3), zero_cnn=True)
    st = O.fdcnn_forward(inp["s"], inp["params"], cfg.chans, cfg.N_d)
    assert np.array_equal(st, inp["s"].astype(np.complex128))


def _torch_reference(s, params, chans, N_d):
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    n, U, _ = s.shape
    S = int(np.ceil(np.sqrt(N_d)))
    flat = np.zeros((n * U, S * S), complex)
    flat[:, :N_d] = s.reshape(n * U, N_d)
    img = flat.reshape(n * U, S, S)
    h = torch.tensor(np.stack([img.real, img.imag], 1), dtype=torch.float64)
    off = 0
    for layer, (ci, co) in enumerate(zip(chans[:-1], chans[1:])):
        W = torch.tensor(params[off:off + co * ci * 9].reshape(co, ci, 3, 3), dtype=torch.float64)
        off += co * ci * 9
        b = torch.tensor(params[off:off + co], dtype=torch.float64)
        off += co
        h = F.conv2d(h, W, b, padding=1)
        if layer < len(chans) - 2:
            h = torch.tanh(h)
    h = h.numpy()
    r = (h[:, 0] + 1j * h[:, 1]).reshape(n * U, S * S)[:, :N_d].reshape(n, U, N_d)
    return s + r


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_fdcnn_vs_torch_conv2d_float64(name):
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(2))
    s = inp["s"].astype(np.complex128)
    p = inp["params"].astype(np.float64)
    got = O.fdcnn_forward(s, p, cfg.chans, cfg.N_d)
    want = _torch_reference(s, p, cfg.chans, cfg.N_d)
    assert np.max(np.abs(got - want)) < 1e-12


def test_fdcnn_brute_force_loops_c1():
    cfg = configs.C1
    inp = gen.make_inputs(cfg, range(1))
    s = inp["s"].astype(np.complex128)
    p = inp["params"].astype(np.float64)
    S, Nd = cfg.S, cfg.N_d
    want = np.empty_like(s)
    for u in range(cfg.U):
        h = [[[0.0] * S for _ in range(S)] for _ in range(2)]
        for i in range(Nd):
            h[0][i // S][i % S] = s[0, u, i].real
            h[1][i // S][i % S] = s[0, u, i].imag
        off = 0
        for layer, (ci, co) in enumerate(zip(cfg.chans[:-1], cfg.chans[1:])):
            W = p[off:off + co * ci * 9]
            off += co * ci * 9
            b = p[off:off + co]
            off += co
            out = [[[0.0] * S for _ in range(S)] for _ in range(co)]
            for o in range(co):
                for y in range(S):
                    for x in range(S):
                        acc = b[o]
                        for c in range(ci):
                            for dy in range(3):
                                for dx in range(3):
                                    yy, xx = y + dy - 1, x + dx - 1
                                    if 0 <= yy < S and 0 <= xx < S:
                                        acc += W[((o * ci + c) * 3 + dy) * 3 + dx] * h[c][yy][xx]
                        out[o][y][x] = np.tanh(acc) if layer < cfg.n_layers - 1 else acc
            h = out
        for i in range(Nd):
            want[0, u, i] = s[0, u, i] + h[0][i // S][i % S] + 1j * h[1][i // S][i % S]
    assert np.max(np.abs(O.fdcnn_forward(s, p, cfg.chans, Nd) - want)) < 1e-13


def test_fdcnn_centre_tap_closed_form():
    rng = np.random.default_rng(3)
    W = np.zeros((2, 2, 3, 3))
    A = rng.standard_normal((2, 2))
    W[:, :, 1, 1] = A
    b = rng.standard_normal(2)
    s = _crandn(rng, 2, 3, 50)
    got = O.fdcnn_forward(s, np.concatenate([W.ravel(), b]), (2, 2), 50)
    re = A[0, 0] * s.real + A[0, 1] * s.imag + b[0]
    im = A[1, 0] * s.real + A[1, 1] * s.imag + b[1]
    assert np.max(np.abs(got - (s + re + 1j * im))) < 1e-13


def test_fdcnn_ue_independence():
    cfg = configs.C2
    inp = gen.make_inputs(cfg, range(1))
    s = inp["s"].astype(np.complex128)
    a = O.fdcnn_forward(s, inp["params"], cfg.chans, cfg.N_d)
    s2 = s.copy()
    s2[0, 1:] = 0.3 - 0.2j
    b = O.fdcnn_forward(s2, inp["params"], cfg.chans, cfg.N_d)
    assert np.array_equal(a[0, 0], b[0, 0]) and not np.allclose(a[0, 1], b[0, 1])


# ============================================================================ channel / ZF
def test_channel_fd_single_tap_and_brute_force():
    rng = np.random.default_rng(4)
    h = _crandn(rng, 1, 2, 8)
    Hfd = O.channel_fd(h, 128, 36)
    assert np.max(np.abs(Hfd - h[0][None])) < 1e-15        # T = 1: flat channel
    h = _crandn(rng, 4, 2, 8)
    Hfd = O.channel_fd(h, 128, 36)
    for j in (0, 17, 18, 35):
        k = (j - 18) % 128
        ref = sum(h[t] * np.exp(-2j * np.pi * k * t / 128) for t in range(4))
        assert np.max(np.abs(Hfd[j] - ref)) < 1e-14


def test_zf_spec_examples_and_pinv():
    # H = [1, 0] -> [1, 0]^T ; H = 2I -> 0.5 I (unnormalised P0)
    _, _, P0 = O.zf_precoder(np.array([[[1.0, 0.0]]]), 1, 1.0)
    assert np.allclose(P0[0], [[1.0], [0.0]])
    _, _, P0 = O.zf_precoder(2 * np.eye(2)[None], 1, 1.0)
    assert np.allclose(P0[0], 0.5 * np.eye(2))
    rng = np.random.default_rng(6)
    H = _crandn(rng, 20, 4, 16)
    P, alpha, P0 = O.zf_precoder(H, 256, 0.3)
    for j in range(20):
        assert np.max(np.abs(H[j] @ P0[j] - np.eye(4))) < 1e-12
        assert np.max(np.abs(P0[j] - np.linalg.pinv(H[j]))) < 1e-12     # SVD route
        assert np.max(np.abs(H[j] @ P[j] - alpha * np.eye(4))) < 1e-11
    assert np.allclose(P, alpha * P0)


def test_zf_alpha_sets_td_rms_statistically():
    """Reading A12: mean over antennas, samples and symbols of |x|^2 = rho^2 (E|s|^2 = 1)."""
    cfg = configs.ChainConfig("t", U=2, B=8, N_fft=64, N_d=36, os=2, M_qam=16, n_sym=3000, T=4,
                              pdp="uniform", orders=(1,), L=0, M=0, chans=(2, 2), spread=0.0, seed=11)
    inp = gen.make_inputs(cfg)
    Hfd = O.channel_fd(inp["h_taps"], cfg.N_ifft, cfg.N_d)
    P, alpha, _ = O.zf_precoder(Hfd, cfg.N_ifft, cfg.rho)
    x = O.ofdm_modulate(O.precode(P, inp["s"]), cfg.N_ifft)
    rms = np.sqrt(np.mean(np.abs(x) ** 2))
    assert abs(rms / cfg.rho - 1.0) < 0.01


# ============================================================================ GMP
def test_gmp_golden_hand_expanded():
    g = _read_golden("gmp_3sample.txt")
    y = O.gmp_pa(g["u"][None, None, :], g["coef"][None, :], (1, 3), 1, 1)
    assert np.max(np.abs(y[0, 0] - g["y"])) < 1e-14


def test_gmp_special_cases():
    rng = np.random.default_rng(7)
    u = 0.3 * _crandn(rng, 2, 3, 64)
    orders, L, M = (1, 3, 5), 2, 1
    n = len(orders) * (L + 1) + 2 * (len(orders) - 1) * (L + 1) * M
    c = np.zeros((3, n), complex)
    c[:, 0] = 1
    assert np.array_equal(O.gmp_pa(u, c, orders, L, M), u)                 # identity PA
    assert np.array_equal(O.gmp_pa(0 * u, _crandn(rng, 3, n), orders, L, M), 0 * u)
    a3 = -0.08 + 0.02j
    c = np.zeros((3, n), complex)
    c[:, 0] = 1
    c[:, L + 1] = a3                                                        # a_{3,0}
    assert np.max(np.abs(O.gmp_pa(u, c, orders, L, M) - (u + a3 * u * np.abs(u) ** 2))) < 1e-15


def test_gmp_linear_terms_are_lti_filter():
    """Only a_{1,l}: y = sum_l a_{1,l} u_{n-l} (circular) -> DFT(y)_k = A(k) DFT(u)_k with
    A(k) = sum_l a_{1,l} e^{-j 2 pi k l / N}.  Pins lag direction and wrap."""
    rng = np.random.default_rng(8)
    N, L, M, orders = 128, 4, 2, (1, 3)
    n = 2 * (L + 1) + 2 * (L + 1) * M
    c = np.zeros((1, n), complex)
    c[0, :L + 1] = _crandn(rng, L + 1)
    u = _crandn(rng, 1, 1, N)
    y = O.gmp_pa(u, c, orders, L, M)
    k = np.arange(N)
    A = sum(c[0, l] * np.exp(-2j * np.pi * k * l / N) for l in range(L + 1))
    assert np.max(np.abs(np.fft.fft(y[0, 0]) - A * np.fft.fft(u[0, 0]))) < 1e-11


def test_gmp_cross_term_direction():
    """b uses the lagging envelope |u_{n-l-g}|, c the leading one |u_{n-l+g}| (Eq. 9)."""
    N = 16
    u = np.zeros((1, 1, N), complex)
    u[0, 0, :] = 1.0
    u[0, 0, 5] = 2.0                         # |u_5|^2 = 4, all others 1
    orders, L, M = (1, 3), 0, 1
    c = np.zeros((1, 4), complex)            # a10 a30 | b301 | c301
    c[0, 2] = 1.0                            # b only: y_n = u_n |u_{n-1}|^2
    y = O.gmp_pa(u, c, orders, L, M)[0, 0]
    assert y[6] == 4.0 and y[4] == 1.0 and y[5] == 2.0
    c = np.zeros((1, 4), complex)
    c[0, 3] = 1.0                            # c only: y_n = u_n |u_{n+1}|^2
    y = O.gmp_pa(u, c, orders, L, M)[0, 0]
    assert y[4] == 4.0 and y[6] == 1.0 and y[5] == 2.0


def test_gmp_linear_in_coefficients():
    rng = np.random.default_rng(9)
    cfg = configs.C2
    u = 0.3 * _crandn(rng, 1, 2, 256)
    c1, c2 = _crandn(rng, 2, cfg.n_coef), _crandn(rng, 2, cfg.n_coef)
    f = lambda c: O.gmp_pa(u, c, cfg.orders, cfg.L, cfg.M)
    assert np.max(np.abs(f(c1 + 2.5 * c2) - f(c1) - 2.5 * f(c2))) < 1e-12


# ============================================================================ receive / chain
def test_receive_fd_equals_td_channel_then_dft():
    """Eq. (3) (circular TD convolution) followed by the DFT equals Eq. (4)/(5)."""
    cfg = configs.C1
    rng = np.random.default_rng(10)
    y = _crandn(rng, 2, cfg.B, cfg.N_ifft)
    h = gen.channel_taps(cfg)
    r = O.channel_td(y, h)
    want = np.fft.fft(r, axis=-1, norm="ortho")[..., O.data_bins(cfg.N_d, cfg.N_ifft)]
    got = O.ue_receive(y, O.channel_fd(h, cfg.N_ifft, cfg.N_d), cfg.N_d)
    assert np.max(np.abs(got - want)) < 1e-12


@pytest.mark.parametrize("name,nsym", [("C1", 4), ("C2", 2)])
def test_end_to_end_invariant_zero_cnn_linear_pa(name, nsym):
    """North-star invariant: zero-weight CNN + linear PA + noiseless ZF => z = s, SER = 0."""
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(nsym), zero_cnn=True, linear_pa=True)
    out = O.run_config(cfg, inp)
    z = out["yhat"] / out["alpha"]
    assert np.max(np.abs(z - inp["s"])) < 1e-12
    assert out["counts"][0] == 0 and out["counts"][1] == nsym * cfg.U * cfg.N_d


def test_full_chain_c1_runs_and_is_sane():
    cfg = configs.C1
    out = O.run_config(cfg, gen.make_inputs(cfg))
    assert out["counts"][1] == cfg.n_sym * cfg.U * cfg.N_d
    assert 0 <= out["counts"][0] <= out["counts"][1]
    rms = np.sqrt(np.mean(np.abs(out["x"]) ** 2))
    assert 0.2 < rms < 0.4


# ============================================================================ paper FD-CNN head (NEXT f2)
def test_fdcnn_paper_golden_hand_computed():
    g = _read_golden("fdcnn_paper_2x2.txt")
    W1 = np.zeros((1, 2, 3, 3))
    W1[0, 0, 1, 1] = 1.0
    W1[0, 1, 0, 0] = 2.0
    W2 = np.array([[1, 0, 1, 0], [2, 0, -1, 0], [-1, 0, 0, 0], [0, 0, 0.5, 0]], dtype=float)
    params = np.concatenate([W1.ravel(), [0.5], W2.ravel(), [0.1, 0.2, 0.3, 0.4]])
    st = O.fdcnn_paper_forward(g["s"][None, None, :], params, 2, n_conv=1)
    assert np.max(np.abs(st[0, 0] - g["st"])) < 1e-14


def test_fdcnn_paper_vs_torch_float64():
    torch = pytest.importorskip("torch")
    F = torch.nn.functional
    cfg = configs.PAPER
    inp = gen.make_inputs(cfg, range(2))
    s = inp["s"].astype(np.complex128)
    p = inp["params"].astype(np.float64)
    S, Nd, nc = cfg.S, cfg.N_d, cfg.n_conv
    K = nc * S * S
    W1 = torch.tensor(p[:nc * 18].reshape(nc, 2, 3, 3))
    b1 = torch.tensor(p[nc * 18:nc * 19])
    W2 = torch.tensor(p[nc * 19:nc * 19 + 2 * Nd * K].reshape(2 * Nd, K))
    b2 = torch.tensor(p[nc * 19 + 2 * Nd * K:])
    flat = np.zeros((s.shape[0] * cfg.U, S * S), complex)
    flat[:, :Nd] = s.reshape(-1, Nd)
    img = torch.tensor(np.stack([flat.real, flat.imag], 1).reshape(-1, 2, S, S))
    out = F.linear(torch.relu(F.conv2d(img, W1, b1, padding=1)).flatten(1), W2, b2).numpy()
    want = (out[:, :Nd] + 1j * out[:, Nd:]).reshape(s.shape)
    assert np.max(np.abs(O.fdcnn_paper_forward(s, p, Nd, nc) - want)) < 1e-12


def test_fdcnn_paper_identity_head_and_chain_invariant():
    cfg = configs.PAPER
    inp = gen.make_inputs(cfg, range(2), zero_cnn=True, linear_pa=True)
    st = O.fdcnn_paper_forward(inp["s"], inp["params"], cfg.N_d, cfg.n_conv)
    assert np.max(np.abs(st - inp["s"])) < 1e-12
    out = O.run_config(cfg, inp)
    assert np.max(np.abs(out["yhat"] / out["alpha"] - inp["s"])) < 1e-12 and out["counts"][0] == 0


def test_paper_flop_formula_eqs_16_18():
    """C_Conv = 2 N^Conv L_U (2 K_C^2 - 1) (S/K_S)^2, C_FC = 8 N_d L_U (S/K_S)^2:
    1,256,000 at the paper's N_d = 384 (S = 20); Fig. 3 prints 1,205,760 = the same with
    S^2 -> N_d (reading A23).  Counts the MACs the oracle's head performs (x2 FLOP)."""
    Nd, S, nc = 384, 20, 2
    conv = 2 * nc * 1 * (2 * 9 - 1) * S * S
    fc = 8 * Nd * 1 * S * S
    assert conv + fc == 1_256_000
    assert 2 * nc * (2 * 9 - 1) * Nd + 8 * Nd * Nd == 1_205_760
    # the oracle's FC is a (2 N_d) x (N^Conv S^2) matrix: 2 * MACs == C_FC
    assert 2 * (2 * Nd) * (nc * S * S) == fc

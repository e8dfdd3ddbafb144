"""GPU parity: every stage of the CUDA path (through the C ABI) against the fp64
oracle on the same seeded inputs.  Bar (north star): relative L2 <= 2e-5 per stage
output; symbol decisions identical except where the oracle's sample lies within
1e-4 of a slicing boundary; integer counts exact under that rule."""
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
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def dev(x, dtype=torch.complex64):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def host(t):
    return t.cpu().numpy()


def crandn(rng, *shape, scale=1.0):
    return (scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))).astype(np.complex64)


# ============================================================================ a4 / FFT
@pytest.mark.parametrize("N,Nd", [(16, 8), (32, 20), (64, 64), (128, 36), (256, 100), (512, 300), (1024, 600),
                                  (2048, 1200), (4096, 600), (8192, 1200), (16384, 3300), (4096, 384), (256, 20),
                                  (256, 34), (16384, 16384)])
def test_ofdm_modulate(F, N, Nd):
    rng = np.random.default_rng(N)
    X = crandn(rng, 3, 5, Nd)
    got = host(F.ofdm_modulate(dev(X), N))
    assert rel(got, O.ofdm_modulate(X, N)) < 2e-6


def test_ofdm_vs_brute_force_small(F):
    rng = np.random.default_rng(0)
    N, Nd = 64, 36
    X = crandn(rng, 1, 2, Nd)
    full = np.zeros((1, 2, N), complex)
    full[..., O.data_bins(Nd, N)] = X
    n = np.arange(N)
    brute = full @ (np.exp(2j * np.pi * np.outer(n, n) / N) / np.sqrt(N)).T
    assert rel(host(F.ofdm_modulate(dev(X), N)), brute) < 2e-6


# ============================================================================ a5 / GMP
GMP_CASES = [((1, 3, 5), 2, 1), ((1, 3, 5, 7), 4, 2), ((1, 3, 5, 7, 9), 6, 3), ((1, 3, 5, 7), 3, 1),  # specialised
             ((1, 5, 9), 3, 0), ((1, 3), 1, 1), ((1,), 0, 0), ((1, 3, 5, 7, 9, 11), 2, 2)]  # generic


@pytest.mark.parametrize("orders,L,M", GMP_CASES)
@pytest.mark.parametrize("N", [128, 4096])
def test_gmp_pa(F, orders, L, M, N):
    rng = np.random.default_rng(L * 10 + M)
    Kp = len(orders)
    ncoef = Kp * (L + 1) + 2 * (Kp - 1) * (L + 1) * M
    x = crandn(rng, 2, 3, N, scale=0.3 / np.sqrt(2))
    coef = crandn(rng, 3, ncoef, scale=0.1)
    coef[:, 0] = 1.0
    got = host(F.gmp_pa(dev(x), dev(coef), orders, L, M))
    assert rel(got, O.gmp_pa(x, coef, orders, L, M)) < TOL


def test_gmp_golden_3sample_wrap(F):
    # N must be >= 16 on the GPU: embed the hand-expanded case of tests/golden/gmp_3sample.txt
    # is impossible (N = 3); instead check the GPU on the oracle at the smallest N with full wrap.
    rng = np.random.default_rng(3)
    x = crandn(rng, 1, 1, 16)
    coef = crandn(rng, 1, 8)
    got = host(F.gmp_pa(dev(x), dev(coef), (1, 3), 1, 1))
    assert rel(got, O.gmp_pa(x, coef, (1, 3), 1, 1)) < TOL


# ============================================================================ a1 / CNN
@pytest.mark.parametrize("name,nsym", [("C1", 4), ("C2", 6), ("C3", 2), ("C4", 1), ("C5", 1)])
def test_fdcnn_forward(F, name, nsym):
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(nsym))
    got = host(F.fdcnn_forward(dev(inp["params"], torch.float32), cfg.chans, dev(inp["s"])))
    want = O.fdcnn_forward(inp["s"], inp["params"], cfg.chans, cfg.N_d)
    assert rel(got, want) < TOL
    assert rel(got - inp["s"], want - inp["s"]) < 1e-4       # the residual itself


@pytest.fixture
def cnn_path(F):
    def set_path(p):
        F.set_cnn_path(p)
        F.set_cnn_tc_precision(0)

    def set_named(name):
        """simt | tensor (FP16-split hidden layers, ACT16 activations) | tensor_tf32 (TF32 split)."""
        set_path(F.CNN_SIMT if name == "simt" else F.CNN_TENSOR)
        if name == "tensor_tf32":
            F.set_cnn_tc_precision(1)

    set_path.named = set_named
    yield set_path
    F.set_cnn_path(F.CNN_AUTO)
    F.set_cnn_tc_precision(0)


@pytest.mark.parametrize("path", ["simt", "tensor", "tensor_tf32"])
@pytest.mark.parametrize("chans,N_d,nsym,U", [((2, 16, 16, 2), 600, 37, 4),      # C2 shape, many tiles / CTA
                                             ((2, 32, 32, 32, 2), 1200, 3, 8),  # C3
                                             ((2, 64, 64, 64, 64, 2), 3300, 1, 4),  # C5 widths (streamed W)
                                             ((2, 16, 32, 64, 2), 500, 5, 3),    # mixed widths, ragged S
                                             ((2, 16, 2), 37, 9, 2),             # no hidden-to-hidden layer, S = 7
                                             ((2, 32, 2), 2, 4, 1)])             # S = 2: one partial tile
def test_fdcnn_paths(F, cnn_path, path, chans, N_d, nsym, U):
    """Tensor-core (FP16 / TF32 split tcgen05) and SIMT FD-CNN paths against the fp64 oracle."""
    cnn_path.named(path)
    rng = np.random.default_rng(len(chans) * 1000 + N_d)
    s = crandn(rng, nsym, U, N_d, scale=0.7)
    n_par = sum(co * ci * 9 + co for ci, co in zip(chans[:-1], chans[1:]))
    params = (0.05 * rng.standard_normal(n_par)).astype(np.float32)
    got = host(F.fdcnn_forward(dev(params, torch.float32), chans, dev(s)))
    want = O.fdcnn_forward(s, params, chans, N_d)
    assert rel(got, want) < TOL
    assert rel(got - s, want - s) < 1e-4


@pytest.mark.parametrize("path", ["simt", "tensor", "tensor_tf32"])
@pytest.mark.parametrize("seed", range(8))
def test_fdcnn_random_shapes(F, cnn_path, path, seed):
    """Seeded random networks / image sizes on both CNN paths (tensor path: hidden widths in
    {16, 32, 64}; SIMT path: any width) against the fp64 oracle."""
    rng = np.random.default_rng(7000 + seed)
    depth = int(rng.integers(1, 5))
    widths = [16, 32, 64] if path != "simt" else [3, 8, 16, 20, 32]
    chans = (2,) + tuple(int(rng.choice(widths)) for _ in range(depth)) + (2,)
    N_d = 2 * int(rng.integers(1, 300))
    U, nsym = int(rng.integers(1, 5)), int(rng.integers(1, 4))
    cnn_path.named(path)
    s = crandn(rng, nsym, U, N_d, scale=0.7)
    n_par = sum(co * ci * 9 + co for ci, co in zip(chans[:-1], chans[1:]))
    params = (0.05 * rng.standard_normal(n_par)).astype(np.float32)
    got = host(F.fdcnn_forward(dev(params, torch.float32), chans, dev(s)))
    want = O.fdcnn_forward(s, params, chans, N_d)
    assert rel(got, want) < TOL, (chans, N_d, U, nsym)


def test_fdcnn_tensor_full_batch_sampled(F, cnn_path):
    """C2 at the bench batch (1024 symbols) on the tensor-core path; the oracle checks
    sampled symbols one by one (the CNN acts per symbol image)."""
    cfg = configs.C2
    cnn_path(F.CNN_TENSOR)
    inp = gen.make_inputs(cfg, range(cfg.n_sym))
    got = host(F.fdcnn_forward(dev(inp["params"], torch.float32), cfg.chans, dev(inp["s"])))
    for n in (0, 1, 511, 1023):
        want = O.fdcnn_forward(inp["s"][n:n + 1], inp["params"], cfg.chans, cfg.N_d)
        assert rel(got[n:n + 1], want) < TOL


@pytest.mark.parametrize("nsym", [1, 3, 40])
def test_fdcnn_paper_forward(F, nsym):
    """Paper FD-CNN head (NEXT f2): conv + ReLU + FC GEMM vs the oracle; ragged M, N tails."""
    cfg = configs.PAPER
    inp = gen.make_inputs(cfg, range(nsym))
    got = host(F.fdcnn_paper_forward(dev(inp["params"], torch.float32), cfg.n_conv, dev(inp["s"])))
    want = O.fdcnn_paper_forward(inp["s"], inp["params"], cfg.N_d, cfg.n_conv)
    assert rel(got, want) < TOL


def test_fdcnn_paper_identity_head(F):
    cfg = configs.PAPER
    inp = gen.make_inputs(cfg, range(5), zero_cnn=True)
    got = host(F.fdcnn_paper_forward(dev(inp["params"], torch.float32), cfg.n_conv, dev(inp["s"])))
    assert rel(got, inp["s"]) < 2e-6


def test_fdcnn_zero_weights_identity(F):
    cfg = configs.C2
    inp = gen.make_inputs(cfg, range(3), zero_cnn=True)
    got = host(F.fdcnn_forward(dev(inp["params"], torch.float32), cfg.chans, dev(inp["s"])))
    assert np.array_equal(got, inp["s"])


# ============================================================================ a2 / ZF
@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C5"])
def test_zf_precoder_build(F, name):
    cfg = configs.get(name)
    h = gen.channel_taps(cfg)
    h_fd, P, alpha = F.zf_precoder_build(dev(h), cfg.N_ifft, cfg.N_d, cfg.rho)
    Hfd = O.channel_fd(h, cfg.N_ifft, cfg.N_d)
    Po, ao, _ = O.zf_precoder(Hfd, cfg.N_ifft, cfg.rho)
    assert rel(host(h_fd), Hfd.transpose(1, 2, 0)) < TOL
    assert rel(host(P), Po.transpose(1, 2, 0)) < TOL
    assert abs(alpha / ao - 1) < 1e-6


def test_zf_antenna_rows(F):
    cfg = configs.C2
    h = gen.channel_taps(cfg)
    _, Pfull, a = F.zf_precoder_build(dev(h), cfg.N_ifft, cfg.N_d, cfg.rho)
    _, Pl, al = F.zf_precoder_build(dev(h), cfg.N_ifft, cfg.N_d, cfg.rho, b0=16, B_loc=16)
    assert al == a and torch.equal(Pl, Pfull[16:32])


# ============================================================================ a3 / precode, fused tx
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_precode(F, name):
    cfg = configs.get(name)
    rng = np.random.default_rng(1)
    P = crandn(rng, cfg.B, cfg.U, cfg.N_d)
    s = crandn(rng, 3, cfg.U, cfg.N_d)
    got = host(F.precode(dev(P), dev(s)))
    assert rel(got, O.precode(P.transpose(2, 0, 1), s)) < TOL


@pytest.mark.parametrize("n,B,U,Nd", [(11, 512, 32, 3300), (9, 37, 5, 70), (1, 8, 2, 36), (17, 256, 16, 3300),
                                      (64, 64, 4, 600)])
def test_precode_tiles_ragged(F, n, B, U, Nd):
    """Tiled precode over ragged symbol / antenna / subcarrier tiles (NT = 8, 4 antennas per
    thread, 32 subcarriers per CTA) against the oracle contraction."""
    rng = np.random.default_rng(n * 7 + B)
    P = crandn(rng, B, U, Nd)
    s = crandn(rng, n, U, Nd)
    got = host(F.precode(dev(P), dev(s)))
    assert got.shape == (n, B, Nd)
    assert rel(got, O.precode(P.transpose(2, 0, 1), s)) < TOL


@pytest.mark.parametrize("n,B,U,Nd", [(11, 512, 32, 3300), (9, 37, 12, 70), (17, 256, 16, 600), (3, 64, 4, 600),
                                      (5, 40, 7, 36), (2, 24, 24, 100), (25, 37, 20, 3302), (41, 19, 13, 1998)])
def test_combine_ser_ragged(F, n, B, U, Nd):
    """Channel sum + slicing (register-blocked kernel for U <= 8, staged tile kernel for
    U = 9..32) on ragged symbol / subcarrier / antenna counts against the oracle einsum and
    slicer; decisions identical except within 1e-4 of a boundary.  The last two shapes have more
    tiles than a B200 holds CTAs (296), so whole tiles and the half tiles of the last round run in
    one launch, with a one-symbol last tile (an empty second half), an odd antenna count (a
    partial last stage), a subcarrier count off the 32-wide tiles and unused user lanes."""
    rng = np.random.default_rng(n * 131 + U)
    M_qam = 64
    XPA = crandn(rng, n, B, Nd, scale=0.3)
    h = crandn(rng, U, B, Nd, scale=0.3)
    alpha = 0.7
    idx = rng.integers(0, M_qam, size=(n, U, Nd)).astype(np.uint16)
    want = np.einsum("ubj,nbj->nuj", h.astype(np.complex128), XPA.astype(np.complex128))
    d_idx = torch.from_numpy(idx.astype(np.int32)).to("cuda").to(torch.uint16)
    dec = torch.zeros((n, U, Nd), dtype=torch.uint16, device="cuda")
    yhat, counts, _ = F.ue_combine_ser(dev(XPA), dev(h), alpha, d_idx, M_qam, dec=dec)
    assert rel(host(yhat), want) < TOL
    assert rel(host(F.ue_combine(dev(XPA), dev(h))), want) < TOL
    dec_o, c_o = O.slice_ser(want, alpha, idx, M_qam)
    _, near = _near_mask(want, alpha, M_qam)
    dg = host(dec)
    assert np.array_equal(dg[~near], dec_o[~near])          # element by element outside the 1e-4 band
    c = host(counts)
    assert c[1] == n * U * Nd
    err_gpu = int((dg != idx).sum())
    assert c[0] == err_gpu
    assert abs(err_gpu - int(c_o[0])) <= int(near.sum())


@pytest.mark.parametrize("ws,nm,B,U,Nd", [(1, 5, 24, 16, 200), (3, 4, 30, 32, 132), (2, 40, 9, 12, 1300), (8, 1, 64, 32, 70)])
def test_combine_peer_exchange(F, ws, nm, B, U, Nd):
    """Mode A's fused exchange on one GPU: `ws` ranks run one after the other, each with its
    antenna shard of the world batch, ue_combine_peer storing the partial sums into the owners'
    receive buffers (all local here); every owner's ue_reduce_ser must then equal the oracle's
    full channel sum over all antennas (Eq. 5) on its own symbols, decisions element by
    element outside the 1e-4 band, and untouched slots stay as they were."""
    from paper_2205_05158_b200 import dist as D
    rng = np.random.default_rng(ws * 17 + U)
    M_qam, alpha, n = 16, 0.9, ws * nm
    XPA = crandn(rng, n, B, Nd, scale=0.3)
    h = crandn(rng, U, B, Nd, scale=0.3)
    idx = rng.integers(0, M_qam, size=(n, U, Nd)).astype(np.uint16)
    want = np.einsum("ubj,nbj->nuj", h.astype(np.complex128), XPA.astype(np.complex128))
    recv = [torch.full((ws, nm, U, Nd), 7.0 + 3.0j, dtype=torch.complex64, device="cuda") for _ in range(ws)]
    for r in range(ws):
        b0, bl = D.antenna_shard(B, ws, r)
        F.ue_combine_peer(dev(XPA[:, b0:b0 + bl]), dev(h[:, b0:b0 + bl]), recv, r)
    torch.cuda.synchronize()
    for owner in range(ws):
        got = host(recv[owner])
        for r in range(ws):                                   # slot r holds rank r's partial of the owner's symbols
            b0, bl = D.antenna_shard(B, ws, r)
            part = np.einsum("ubj,nbj->nuj", h[:, b0:b0 + bl].astype(np.complex128),
                             XPA[owner * nm:(owner + 1) * nm, b0:b0 + bl].astype(np.complex128))
            assert rel(got[r], part) < TOL
            assert D.peer_slot(owner * nm + nm - 1, nm, r) == (owner, r, nm - 1)
        sl = slice(owner * nm, (owner + 1) * nm)
        d_idx = torch.from_numpy(idx[sl].astype(np.int32)).to("cuda").to(torch.uint16)
        dec = torch.zeros((nm, U, Nd), dtype=torch.uint16, device="cuda")
        yhat, counts, _ = F.ue_reduce_ser(recv[owner], alpha, d_idx, M_qam, dec=dec)
        assert rel(host(yhat), want[sl]) < TOL
        s_slots = host(recv[owner]).astype(np.complex128).sum(axis=0)       # rank order, like the kernel (fp32 there)
        assert rel(host(yhat), s_slots) < 1e-6
        dec_o, c_o = O.slice_ser(want[sl], alpha, idx[sl], M_qam)
        _, near = _near_mask(want[sl], alpha, M_qam)
        dg = host(dec)
        assert np.array_equal(dg[~near], dec_o[~near])
        c = host(counts)
        assert c[1] == nm * U * Nd and c[0] == int((dg != idx[sl]).sum())
    y2, c2, _ = F.ue_reduce_ser(recv[0])                      # no slicing: counts untouched / absent
    assert c2 is None and rel(host(y2), want[:nm]) < TOL


def test_combine_unaligned_bases(F):
    """XPA / h_fd whose bases are 8- but not 16-byte aligned (views one complex64 into a buffer):
    the tile kernel's 16-byte copies do not apply, the register-blocked kernel takes over."""
    rng = np.random.default_rng(77)
    n, B, U, Nd = 9, 24, 16, 200
    XPA = crandn(rng, n, B, Nd, scale=0.3)
    h = crandn(rng, U, B, Nd, scale=0.3)
    want = np.einsum("ubj,nbj->nuj", h.astype(np.complex128), XPA.astype(np.complex128))
    bx = torch.zeros(XPA.size + 1, dtype=torch.complex64, device="cuda")
    bh = torch.zeros(h.size + 1, dtype=torch.complex64, device="cuda")
    bx[1:] = dev(XPA).reshape(-1)
    bh[1:] = dev(h).reshape(-1)
    Xv, hv = bx[1:].view(n, B, Nd), bh[1:].view(U, B, Nd)
    assert Xv.data_ptr() % 16 == 8 and hv.data_ptr() % 16 == 8
    assert rel(host(F.ue_combine(Xv, hv)), want) < TOL
    assert rel(host(F.ue_combine(dev(XPA), hv)), want) < TOL


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_chain_tx_vs_oracle_and_unfused(F, name):
    cfg = configs.get(name)
    nsym = 2
    inp = gen.make_inputs(cfg, range(nsym))
    h_fd, P, alpha = F.zf_precoder_build(dev(inp["h_taps"]), cfg.N_ifft, cfg.N_d, cfg.rho)
    s = dev(inp["s"])
    coef = dev(inp["coef"])
    y = F.chain_tx(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    y2 = F.gmp_pa(F.ofdm_modulate(F.precode(P, s), cfg.N_ifft), coef, cfg.orders, cfg.L, cfg.M)
    assert rel(host(y), host(y2)) < 2e-6
    Po = host(P).transpose(2, 0, 1)
    want = O.gmp_pa(O.ofdm_modulate(O.precode(Po, inp["s"]), cfg.N_ifft), inp["coef"], cfg.orders, cfg.L, cfg.M)
    assert rel(host(y), want) < TOL


@pytest.mark.parametrize("name,impair", [("C4", False), ("C5", False), ("C4", True)])
def test_chain_cluster_split_vs_single(F, name, impair):
    """The two-CTA cluster split (N = 16384) against the single-CTA kernel on the same
    inputs: one extra radix-2 step, so rounding-level differences only; per-stage oracle
    parity is covered by the other chain tests (which run the split by default)."""
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(2))
    h_fd, P, alpha = F.zf_precoder_build(dev(inp["h_taps"]), cfg.N_ifft, cfg.N_d, cfg.rho)
    s, coef = dev(inp["s"]), dev(inp["coef"])
    imp = F.make_impairments(0.8, 1e-3, 0.0, 0.0, 77, 0, 0, cfg.B) if impair else None

    def run():
        if imp is None:
            return F.chain_txrx(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
        return F.chain_txrx_ex(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft, imp)

    y_cl, X_cl = run()
    F.set_chain_split(1)
    try:
        y_1, X_1 = run()
    finally:
        F.set_chain_split(0)
    assert rel(host(y_cl), host(y_1)) < 1e-6
    assert rel(host(X_cl), host(X_1)) < 1e-6
    if not impair:
        Po = host(P).transpose(2, 0, 1)
        want = O.gmp_pa(O.ofdm_modulate(O.precode(Po, inp["s"]), cfg.N_ifft), inp["coef"], cfg.orders, cfg.L, cfg.M)
        assert rel(host(y_cl), want) < TOL


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_chain_txrx_vs_unfused(F, name):
    """chain_txrx = chain_tx + the receive FFT of ue_receive, in one kernel; XPA feeds ue_combine."""
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(3))
    h_fd, P, alpha = F.zf_precoder_build(dev(inp["h_taps"]), cfg.N_ifft, cfg.N_d, cfg.rho)
    s, coef = dev(inp["s"]), dev(inp["coef"])
    y, XPA = F.chain_txrx(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    y_ref = F.chain_tx(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    # same arithmetic except the pruned first IDFT pass of chain_txrx (rounding-level)
    assert rel(host(y), host(y_ref)) < 1e-6
    want = np.fft.fft(host(y).astype(np.complex128), axis=-1, norm="ortho")[..., O.data_bins(cfg.N_d, cfg.N_ifft)]
    assert rel(host(XPA), want) < 2e-6
    yhat = F.ue_combine(XPA, h_fd)
    assert rel(host(yhat), host(F.ue_receive(y, h_fd))) < 2e-6


@pytest.mark.parametrize("N,N_d,orders,L,M", [
    (4096, 512, (1, 3, 5, 7), 4, 2),      # h = N/16: one data slot per side (PZ = 1)
    (4096, 514, (1, 3, 5, 7), 4, 2),      # h = N/16 + 1: second slot holds one bin (PZ = 2)
    (4096, 1024, (1, 3, 5, 7), 3, 1),     # h = N/8: the largest pruned case
    (4096, 1026, (1, 3, 5, 7), 4, 2),     # h > N/8: generic passes
    (4096, 384, (1, 3, 5, 7), 3, 1),      # the paper's shape (PZ = 1)
    (8192, 1200, (1, 3, 5, 7), 4, 2),     # N = 2 * 16^3: pruned IDFT pass only
    (16384, 3300, (1, 3, 5, 7, 9), 6, 3)])
def test_chain_txrx_pruned_fft(F, N, N_d, orders, L, M):
    """Pruned radix-16 passes (first IDFT pass, last receive-DFT pass) against the oracle's
    precode -> IDFT -> GMP and the fp64 FFT of the returned waveform at the data bins."""
    rng = np.random.default_rng(N + N_d)
    B, U, n = 3, 2, 2
    Kp = len(orders)
    ncoef = Kp * (L + 1) + 2 * (Kp - 1) * (L + 1) * M
    P = crandn(rng, B, U, N_d, scale=0.5)
    s = crandn(rng, n, U, N_d)
    coef = crandn(rng, B, ncoef, scale=0.05)
    coef[:, 0] = 1.0
    y, XPA = F.chain_txrx(dev(P), dev(s), dev(coef), orders, L, M, N)
    x = O.ofdm_modulate(O.precode(P.transpose(2, 0, 1), s), N)
    assert rel(host(y), O.gmp_pa(x, coef, orders, L, M)) < TOL
    want = np.fft.fft(host(y).astype(np.complex128), axis=-1, norm="ortho")[..., O.data_bins(N_d, N)]
    assert rel(host(XPA), want) < 2e-6


_GMP_SHAPES = [((1, 3, 5), 2, 1), ((1, 3, 5, 7), 4, 2), ((1, 3, 5, 7, 9), 6, 3), ((1, 3, 5, 7), 3, 1), ((1, 5), 2, 1)]


@pytest.mark.parametrize("seed", range(24))
def test_chain_random_shapes(F, seed):
    """Seeded random shapes over every kernel variant (transform sizes 16..16384 incl. the
    cluster split, pruned and generic FFT passes, specialised and generic GMP, ragged U/B):
    fused chain_txrx vs the oracle and the fp64 FFT, chain_txrx_pre(precode) vs chain_txrx,
    and the standalone ofdm_modulate -> gmp_pa vs the fused waveform."""
    rng = np.random.default_rng(1000 + seed)
    N = 1 << int(rng.integers(4, 15))
    N_d = 2 * int(rng.integers(1, N // 2 + 1))
    if seed % 3 == 0:
        N_d = 4 * max(1, N_d // 4)          # N_d % 4 == 0 (cluster-split eligible at N = 16384)
    U = int(rng.integers(1, 9))
    B = int(rng.integers(U, U + 5))
    n = int(rng.integers(1, 3))
    orders, L, M = _GMP_SHAPES[seed % len(_GMP_SHAPES)]
    if L + 2 * M >= N:
        L, M = 1, 0
    Kp = len(orders)
    ncoef = Kp * (L + 1) + 2 * (Kp - 1) * (L + 1) * M
    P = crandn(rng, B, U, N_d, scale=0.5)
    s = crandn(rng, n, U, N_d)
    coef = crandn(rng, B, ncoef, scale=0.05)
    coef[:, 0] = 1.0
    y, XPA = F.chain_txrx(dev(P), dev(s), dev(coef), orders, L, M, N)
    x = O.ofdm_modulate(O.precode(P.transpose(2, 0, 1), s), N)
    assert rel(host(y), O.gmp_pa(x, coef, orders, L, M)) < TOL, (N, N_d, U, B, orders, L, M)
    want = np.fft.fft(host(y).astype(np.complex128), axis=-1, norm="ortho")[..., O.data_bins(N_d, N)]
    assert rel(host(XPA), want) < 2e-6
    X = F.precode(dev(P), dev(s))
    y_pre, XPA_pre = F.chain_txrx_pre(X, dev(coef), orders, L, M, N)
    assert rel(host(y_pre), host(y)) < 1e-6 and rel(host(XPA_pre), host(XPA)) < 1e-6
    y2 = F.gmp_pa(F.ofdm_modulate(X, N), dev(coef), orders, L, M)
    assert rel(host(y2), host(y)) < 1e-6
    h = crandn(rng, U, B, N_d, scale=0.3)                      # standalone receive path
    assert rel(host(F.ue_receive(y, dev(h))), host(F.ue_combine(XPA, dev(h)))) < 2e-6


@pytest.mark.parametrize("orders,L,M", [((1, 5, 9), 3, 0), ((1, 3), 1, 1)])
def test_chain_txrx_generic_gmp(F, orders, L, M):
    cfg = configs.C2
    rng = np.random.default_rng(4)
    Kp = len(orders)
    ncoef = Kp * (L + 1) + 2 * (Kp - 1) * (L + 1) * M
    P = crandn(rng, cfg.B, cfg.U, cfg.N_d, scale=0.05)
    s = crandn(rng, 2, cfg.U, cfg.N_d)
    coef = crandn(rng, cfg.B, ncoef, scale=0.1)
    y, XPA = F.chain_txrx(dev(P), dev(s), dev(coef), orders, L, M, cfg.N_ifft)
    want_y = O.gmp_pa(O.ofdm_modulate(O.precode(P.transpose(2, 0, 1), s), cfg.N_ifft), coef, orders, L, M)
    assert rel(host(y), want_y) < TOL
    want = np.fft.fft(want_y, axis=-1, norm="ortho")[..., O.data_bins(cfg.N_d, cfg.N_ifft)]
    assert rel(host(XPA), want) < TOL


# ============================================================================ a6 / receive + SER
@pytest.mark.parametrize("name", ["C1", "C2"])
def test_ue_receive(F, name):
    cfg = configs.get(name)
    rng = np.random.default_rng(2)
    y = crandn(rng, 3, cfg.B, cfg.N_ifft, scale=0.2)
    hfd = crandn(rng, cfg.U, cfg.B, cfg.N_d)
    got = host(F.ue_receive(dev(y), dev(hfd)))
    assert rel(got, O.ue_receive(y, hfd.transpose(2, 0, 1), cfg.N_d)) < TOL
    acc = F.ue_receive(dev(y), dev(hfd))
    F.ue_receive(dev(y), dev(hfd), out=acc, accumulate=True)
    assert rel(host(acc), 2 * got) < 1e-6


@pytest.mark.parametrize("M", [16, 64, 256])
def test_slicer_decisions(F, M):
    rng = np.random.default_rng(M)
    n, U, Nd = 4, 3, 500
    idx = rng.integers(0, M, (n, U, Nd)).astype(np.uint16)
    alpha = 0.8
    yhat = (alpha * (O.qam_points(idx, M) + 0.3 * crandn(rng, n, U, Nd) / np.sqrt(M))).astype(np.complex64)
    dec_o, cnt_o = O.slice_ser(yhat, alpha, idx, M)
    _, near = _near_mask(yhat, alpha, M)
    dec = torch.zeros((n, U, Nd), dtype=torch.uint16, device="cuda")
    counts, _ = F.ue_slice_ser(dev(yhat), alpha, dev(idx, torch.uint16), M, dec=dec)
    dg = host(dec)
    assert np.array_equal(dg[~near], dec_o[~near])
    c = host(counts)
    assert c[1] == n * U * Nd
    assert abs(int(c[0]) - int(cnt_o[0])) <= int(near.sum())


def _near_mask(yhat, alpha, M, eps=1e-4):
    m = int(round(np.sqrt(M)))
    cst = 1.0 / np.sqrt(2.0 * (M - 1) / 3.0)
    z = np.asarray(yhat, np.complex128) / alpha
    near = np.zeros(z.shape, bool)
    for v in (z.real / cst, z.imag / cst):
        bnd = 2.0 * np.round(v / 2.0)
        near |= (np.abs(v - bnd) < eps / cst) & (np.abs(bnd) <= m - 2)
    return z, near


def _decision_eps(yhat_o, alpha):
    """Decision-parity band (DESIGN reading A25): the north star's 1e-4 for unit-scale z,
    widened to the relative-L2 bar times the RMS of z when the received signal is far beyond
    the constellation (C5: RMS |z| ~ 2300, the PA's coherent peaks dominate yhat)."""
    z = np.asarray(yhat_o, np.complex128) / alpha
    return max(1e-4, TOL * float(np.sqrt(np.mean(np.abs(z) ** 2))))


# ============================================================================ end to end
def _gpu_chain(F, cfg, inp, fused=True):
    from paper_2205_05158_b200.chain import Chain, Shapes
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=len(inp["symbols"]))
    s = dev(inp["s"])
    idx = dev(inp["idx"], torch.uint16)
    dec = torch.zeros(idx.shape, dtype=torch.uint16, device="cuda")
    yhat, counts, _ = ch.step(s, idx, dec=dec, fused=fused)
    torch.cuda.synchronize()
    return ch, host(ch.s_tilde[:s.shape[0]]), host(ch.y[:s.shape[0]]), host(yhat), host(counts), host(dec)


@pytest.mark.parametrize("name,fused", [("C1", True), ("C1", False), ("C2", True), ("C2", False), ("P", True)])
def test_end_to_end(F, name, fused):
    """C1: all 4 symbols.  C2: the full 1024-symbol batch in one call (the bench's
    launch configuration); symbols 0, 517, 1023 compared with the oracle."""
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg)
    ch, st, y, yhat, counts, dec = _gpu_chain(F, cfg, inp, fused=fused)
    pick = list(range(cfg.n_sym)) if cfg.n_sym <= 4 else [0, 517, cfg.n_sym - 1]
    sub = gen.make_inputs(cfg, pick)
    o = O.run_config(cfg, sub)
    assert abs(ch.alpha / o["alpha"] - 1) < 1e-6
    assert rel(st[pick], o["s_tilde"]) < TOL
    assert rel(y[pick], o["y"]) < TOL
    assert rel(yhat[pick], o["yhat"]) < TOL
    _, near = _near_mask(o["yhat"], o["alpha"], cfg.M_qam)
    assert np.array_equal(dec[pick][~near], o["dec"][~near])
    assert counts[1] == cfg.n_sym * cfg.U * cfg.N_d
    err_g = int((dec[pick] != inp["idx"][pick]).sum())          # SER errors of the compared symbols
    assert abs(err_g - int(o["counts"][0])) <= int(near.sum())
    assert counts[0] == int((dec != inp["idx"]).sum())


def _decision_report(name, dec_g, o, eps_band):
    """Decision parity at the north star's fixed 1e-4 band and at the A25 band: every decision
    outside the A25 band is identical; the raw north-star mismatches (outside 1e-4) are
    printed with their boundary distances and must all lie inside the A25 band."""
    cfg = configs.get(name)
    z, near4 = _near_mask(o["yhat"], o["alpha"], cfg.M_qam, 1e-4)
    _, near_b = _near_mask(o["yhat"], o["alpha"], cfg.M_qam, eps_band)
    mism = dec_g != o["dec"]
    raw = mism & ~near4
    cst = 1.0 / np.sqrt(2.0 * (cfg.M_qam - 1) / 3.0)
    dist = []
    for i in np.argwhere(raw):
        zz = z[tuple(i)]
        d = min(abs(v / cst - 2.0 * np.round(v / cst / 2.0)) * cst for v in (zz.real, zz.imag))
        dist.append(float(d))
    print(f"{name}: decisions {mism.size}, mismatches {int(mism.sum())}, outside the north-star 1e-4 band "
          f"{int(raw.sum())} (boundary distances {sorted(dist)[:8]}), A25 band {eps_band:.3g}")
    assert not (mism & ~near_b).any()
    assert int(raw.sum()) <= max(2, mism.size // 10000)


@pytest.mark.parametrize("name,nsym,pick", [("C3", 8, [5]), ("C4", 8, [5]), ("C5", 8, [5]), ("C3", 512, [0, 509]),
                                           ("C4", 128, [0, 125]), ("C5", 32, [3, 29])])
def test_end_to_end_large(F, name, nsym, pick):
    """The large configurations through the whole step on their own paths: tensor-core CNN
    with the FP32 last layer, the precode + chain_txrx_pre (U >= 16), the N = 8192
    256-thread / N = 16384 cluster-split chain, the staged-tile channel sum.  Small batches
    and the bench's batches (C3 512, C4 128, C5 32 symbols per step); one or two symbols of
    the batch (one in the last 8-symbol tile) against the oracle: every stage output at 2e-5,
    decisions (north-star band and A25 band, _decision_report) and the SER error count of the
    compared symbols."""
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(nsym))
    ch, st, y, yhat, counts, dec = _gpu_chain(F, cfg, inp)
    o = O.run_config(cfg, gen.make_inputs(cfg, pick))
    assert abs(ch.alpha / o["alpha"] - 1) < 1e-6
    assert rel(st[pick], o["s_tilde"]) < TOL
    assert rel(y[pick], o["y"]) < TOL
    assert rel(yhat[pick], o["yhat"]) < TOL
    eps_band = _decision_eps(o["yhat"], o["alpha"])
    _decision_report(name, dec[pick], o, eps_band)
    _, near_b = _near_mask(o["yhat"], o["alpha"], cfg.M_qam, eps_band)
    err_g = int((dec[pick] != inp["idx"][pick]).sum())
    assert abs(err_g - int(o["counts"][0])) <= int(near_b.sum())
    assert counts[1] == nsym * cfg.U * cfg.N_d
    assert counts[0] == int((dec != inp["idx"]).sum())


TOL_TF32 = 2e-3          # north star: "<= 2e-3 (TF32 tensor-core precoding)"
EPS_TF32 = 5e-3          # SURVEY §8(c) reading A22: TF32 moves z by ~3e-4, so the band is scaled to 5e-3


@pytest.mark.parametrize("nsym,pick", [(8, [5]), (512, [0, 509])])
def test_end_to_end_c3_tf32_precode(F, nsym, pick):
    """BASELINE configs[2]: C3 with the "TF32 tensor-core precoding variant reported separately"
    (precode on tcgen05 kind::tf32, one pass, then chain_txrx_pre; bench --split-precode
    --precode-math tf32).  Against the fp64 oracle: s_tilde at the FP32 bar (the CNN is
    unchanged), the precoded / PA / received signals at the TF32 bar 2e-3, and decisions
    identical outside the A22 band (5e-3), the mismatches inside it printed with their boundary
    distances (north-star band 1e-4 reported)."""
    from paper_2205_05158_b200.chain import Chain, Shapes
    cfg = configs.C3
    inp = gen.make_inputs(cfg, range(nsym))
    ch = Chain(Shapes.from_config(cfg), inp["h_taps"], inp["coef"], inp["params"], max_batch=nsym,
               precode_math="tf32")
    ch.split_precode = True
    s, idx = dev(inp["s"]), dev(inp["idx"], torch.uint16)
    dec = torch.zeros(idx.shape, dtype=torch.uint16, device="cuda")
    yhat, counts, _ = ch.step(s, idx, dec=dec)
    torch.cuda.synchronize()
    st, X, y, yh, dg, c = (host(ch.s_tilde[:nsym]), host(ch.X[:nsym]), host(ch.y[:nsym]), host(yhat), host(dec),
                           host(counts))
    o = O.run_config(cfg, gen.make_inputs(cfg, pick))
    assert rel(st[pick], o["s_tilde"]) < TOL
    e_X, e_y, e_yh = rel(X[pick], o["X"]), rel(y[pick], o["y"]), rel(yh[pick], o["yhat"])
    print(f"C3 TF32 precode: rel-L2 X {e_X:.2e}, y {e_y:.2e}, yhat {e_yh:.2e}")
    assert 1e-6 < e_X < TOL_TF32                       # TF32 class, not FP32
    assert e_y < TOL_TF32 and e_yh < TOL_TF32
    z, near4 = _near_mask(o["yhat"], o["alpha"], cfg.M_qam, 1e-4)
    _, near_b = _near_mask(o["yhat"], o["alpha"], cfg.M_qam, EPS_TF32)
    mism = dg[pick] != o["dec"]
    cst = 1.0 / np.sqrt(2.0 * (cfg.M_qam - 1) / 3.0)
    dist = sorted(min(abs(v / cst - 2.0 * np.round(v / cst / 2.0)) * cst for v in (z[tuple(i)].real, z[tuple(i)].imag))
                  for i in np.argwhere(mism))
    print(f"C3 TF32 decisions {mism.size}: mismatches {int(mism.sum())} (outside 1e-4: {int((mism & ~near4).sum())}),"
          f" boundary distances {[round(d, 6) for d in dist[:10]]}")
    assert not (mism & ~near_b).any()
    assert c[1] == nsym * cfg.U * cfg.N_d
    assert c[0] == int((dg != inp["idx"]).sum())


@pytest.mark.parametrize("name", ["C1", "C2", "P"])
def test_invariant_zero_cnn_linear_pa(F, name):
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(8 if name == "C2" else 4), zero_cnn=True, linear_pa=True)
    ch, st, y, yhat, counts, dec = _gpu_chain(F, cfg, inp)
    z = yhat / ch.alpha
    assert rel(z, inp["s"]) < TOL
    assert counts[0] == 0 and np.array_equal(dec, inp["idx"])


@pytest.mark.parametrize("name,shards", [("C1", 2), ("C2", 4)])
def test_antenna_shards_accumulate_to_full(F, name, shards):
    """Mode A through the ABI on one GPU: per-shard ZF rows, chain_txrx on the shard's
    antennas and ue_combine(accumulate) over shards == the unsharded received signal."""
    from paper_2205_05158_b200 import dist as D
    cfg = configs.get(name)
    inp = gen.make_inputs(cfg, range(3))
    h, s, coef = dev(inp["h_taps"]), dev(inp["s"]), dev(inp["coef"])
    h_fd, P, _ = F.zf_precoder_build(h, cfg.N_ifft, cfg.N_d, cfg.rho)
    _, XPA = F.chain_txrx(P, s, coef, cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
    full = F.ue_combine(XPA, h_fd)
    acc = torch.zeros_like(full)
    for r in range(shards):
        b0, bl = D.antenna_shard(cfg.B, shards, r)
        hf_r, P_r, _ = F.zf_precoder_build(h, cfg.N_ifft, cfg.N_d, cfg.rho, b0=b0, B_loc=bl)
        _, X_r = F.chain_txrx(P_r, s, coef[b0:b0 + bl].contiguous(), cfg.orders, cfg.L, cfg.M, cfg.N_ifft)
        F.ue_combine(X_r, hf_r, out=acc, accumulate=True)
    assert rel(host(acc), host(full)) < 1e-6


@pytest.mark.parametrize("name", ["C1", "C2", "C4"])
def test_native_runtime_matches(F, name):
    """fd_chain_* (C runtime) == the per-call path; host entry == device entry; oracle counters."""
    from paper_2205_05158_b200.chain import Chain, Shapes
    cfg = configs.get(name)
    nsym = cfg.n_sym if cfg.n_sym <= 4 else (64 if name == "C2" else 8)
    inp = gen.make_inputs(cfg, range(nsym))
    sh = Shapes.from_config(cfg)
    nat = F.NativeChain(sh, inp["h_taps"], inp["coef"], inp["params"], max_batch=nsym)
    ch = Chain(sh, inp["h_taps"], inp["coef"], inp["params"], max_batch=nsym)
    assert nat.alpha == ch.alpha
    s, idx = dev(inp["s"]), dev(inp["idx"], torch.uint16)
    yh_ref, c_ref, _ = ch.step(s, idx)
    yhat = torch.empty_like(yh_ref)
    c_dev = torch.zeros(3, dtype=torch.int64, device="cuda")
    nat.run_device(s, idx, c_dev, yhat=yhat)
    torch.cuda.synchronize()
    assert torch.equal(yhat, yh_ref) and torch.equal(c_dev, c_ref)
    c_host = torch.zeros(3, dtype=torch.int64).pin_memory()
    nat.run_host(torch.from_numpy(inp["s"]).pin_memory(), torch.from_numpy(inp["idx"]).pin_memory(), c_host)
    assert torch.equal(c_host, c_ref.cpu())
    c_q = torch.zeros(3, dtype=torch.int64).pin_memory()
    nat.run_host_qam(torch.from_numpy(inp["idx"]).pin_memory(), c_q)      # device QAM mapping
    assert torch.equal(c_q, c_ref.cpu())
    if name == "C1":
        o = O.run_config(cfg, inp)
        assert c_host[1] == o["counts"][1] and abs(int(c_host[0]) - int(o["counts"][0])) <= int(o["counts"][2])
    with pytest.raises(F.FdpdError):
        nat.run_device(torch.cat([s, s]), torch.cat([idx, idx]), c_dev)     # beyond the plan's batch
    nat.close()


@pytest.mark.parametrize("M", [4, 16, 64, 256])
def test_qam_map_matches_generator(F, M):
    """a0 on the device: bit-identical to the generator's complex64 points (fp64 then round)."""
    rng = np.random.default_rng(M)
    idx = rng.integers(0, M, size=(3, 5, 77)).astype(np.uint16)
    got = host(F.qam_map(torch.from_numpy(idx.astype(np.int32)).cuda().to(torch.uint16), M))
    assert np.array_equal(got.view(np.uint64), gen.qam_symbols(idx, M).view(np.uint64))
    with pytest.raises(F.FdpdError):
        F.qam_map(torch.zeros(4, dtype=torch.uint16, device="cuda"), 12)


# ============================================================================ edge cases / errors
def test_empty_batch_is_noop(F):
    cfg = configs.C1
    x = torch.zeros((0, cfg.B, cfg.N_ifft), dtype=torch.complex64, device="cuda")
    X = torch.zeros((0, cfg.B, cfg.N_d), dtype=torch.complex64, device="cuda")
    assert F.ofdm_modulate(X, cfg.N_ifft).shape == (0, cfg.B, cfg.N_ifft)
    coef = torch.zeros((cfg.B, cfg.n_coef), dtype=torch.complex64, device="cuda")
    assert F.gmp_pa(x, coef, cfg.orders, cfg.L, cfg.M).shape == x.shape


def test_ragged_full_band(F):
    # N_d == N_ifft (no guards), odd symbol count
    rng = np.random.default_rng(9)
    X = crandn(rng, 3, 7, 64)
    assert rel(host(F.ofdm_modulate(dev(X), 64)), O.ofdm_modulate(X, 64)) < 2e-6


def test_argument_errors(F):
    X = torch.zeros((1, 2, 36), dtype=torch.complex64, device="cuda")
    with pytest.raises(F.FdpdError) as e:
        F.ofdm_modulate(X, 100)             # not a power of two
    assert e.value.status == F.FD_ERR_ARG
    with pytest.raises(F.FdpdError):
        F.ofdm_modulate(X, 32)              # N_d > N_ifft
    x = torch.zeros((1, 2, 64), dtype=torch.complex64, device="cuda")
    coef = torch.zeros((2, 4), dtype=torch.complex64, device="cuda")
    with pytest.raises(F.FdpdError):
        F.gmp_pa(x, coef, (1, 2), 1, 1)     # even order
    with pytest.raises(F.FdpdError):
        F.gmp_pa(x, coef, (1, 3), 1, 1, out=x)   # aliasing

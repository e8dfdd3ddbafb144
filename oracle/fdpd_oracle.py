"""fp64 CPU oracle of the FD-CNN DPD downlink chain (arXiv 2205.05158).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2205_05158_b200``) never imports it and the
two share no code: no kernels, helpers, tables or constants.  The only shared
module is ``workload.gen`` (seeded random draws, none of the method's math).

Plain, slow, obviously correct numpy in float64 / complex128.  Each function
follows the paper's definition in the paper's order and notation; PAPER.md
line numbers are cited as P:n, SURVEY.md readings as A<k> (listed in DESIGN.md).

Layouts here are the paper's, not the GPU's:
    s, s_tilde   [n][U][N_d]       (per OFDM symbol, per UE, data subcarrier j)
    Hfd          [N_d][U][B]       (H_hat_k in C^{U x B})
    P            [N_d][B][U]       (P_hat_k in C^{B x U})
    X            [n][B][N_d]       (x_hat_k per antenna at data subcarriers)
    x, y         [n][B][N_ifft]    (time-domain per antenna)
    yhat         [n][U][N_d]

Pins: every function here is checked in tests/test_oracle_*.py against
something other than itself (closed forms, library special cases, brute force,
hand-expanded values).  See DESIGN.md "Parity pins".
"""
from __future__ import annotations

import numpy as np


# ============================================================================ QAM
def qam_points(idx: np.ndarray, M_qam: int) -> np.ndarray:
    """Square M-QAM, unit average energy ("M-QAM constellation").
    Level grid {-(m-1), ..., -1, 1, ..., m-1}; index -> (I = idx mod m, Q = idx div m)
    (reading A19; the labelling is irrelevant for SER).  E|s|^2 = 1 exactly:
    E[l^2] over the m levels is (m^2 - 1)/3 per axis, so c^2 * 2 (M-1)/3 = 1."""
    m = int(round(np.sqrt(M_qam)))
    c = 1.0 / np.sqrt(2.0 * (M_qam - 1) / 3.0)
    lev = np.arange(-(m - 1), m, 2, dtype=np.float64)        # the m odd levels
    idx = np.asarray(idx, dtype=np.int64)
    return (lev[idx % m] + 1j * lev[idx // m]) * c


# ============================================================================ subcarriers
def data_bins(N_d: int, N_ifft: int) -> np.ndarray:
    """IDFT bin of data subcarrier j (reading A7: contiguous, centred, DC included):
    k_j = (j - N_d/2) mod N_ifft, j = 0..N_d-1.  Guards carry P_hat_k = 0."""
    j = np.arange(N_d)
    return (j - N_d // 2) % N_ifft


# ============================================================================ FD-CNN
def fdcnn_forward(s: np.ndarray, params: np.ndarray, chans, N_d: int) -> np.ndarray:
    """FD-CNN DPD, residual conv-stack form (P:167-177 structure; BASELINE network,
    readings A1-A6).

    Per (symbol n, UE u) with L_U = 1:
      * the N_d-vector s[n,u,:] becomes an S x S matrix, S = ceil(sqrt(N_d)), contiguous
        row-major order, zero padding at the tail (P:170 and its footnote);
      * the complex matrix is split into Re and Im channels;
      * layers 1..Lc: h^l[co] = b[co] + sum_ci sum_dy sum_dx W[co,ci,dy,dx] h^{l-1}[ci,y+dy-1,x+dx-1],
        zero outside the image ("zero padding ... same dimension"), tanh after
        every layer but the last (A5);
      * residual output: s_tilde = s + (h^Lc[0] + j h^Lc[1]) cropped to N_d (A5).
    """
    s = np.asarray(s, dtype=np.complex128)
    n, U, nd = s.shape
    assert nd == N_d
    S = int(np.ceil(np.sqrt(N_d)))
    params = np.asarray(params, dtype=np.float64)

    flat = np.zeros((n * U, S * S), dtype=np.complex128)
    flat[:, :N_d] = s.reshape(n * U, N_d)
    img = flat.reshape(n * U, S, S)
    h = np.stack([img.real, img.imag], axis=1)                 # [img][2][S][S]

    off = 0
    n_layers = len(chans) - 1
    for layer in range(n_layers):
        ci_n, co_n = chans[layer], chans[layer + 1]
        W = params[off:off + co_n * ci_n * 9].reshape(co_n, ci_n, 3, 3)
        off += co_n * ci_n * 9
        b = params[off:off + co_n]
        off += co_n
        hp = np.zeros((h.shape[0], ci_n, S + 2, S + 2))
        hp[:, :, 1:S + 1, 1:S + 1] = h
        out = np.broadcast_to(b[None, :, None, None], (h.shape[0], co_n, S, S)).copy()
        for dy in range(3):
            for dx in range(3):
                out += np.einsum("oc,ncyx->noyx", W[:, :, dy, dx],
                                 hp[:, :, dy:dy + S, dx:dx + S])
        h = np.tanh(out) if layer < n_layers - 1 else out
    assert off == params.size
    r = (h[:, 0] + 1j * h[:, 1]).reshape(n * U, S * S)[:, :N_d]
    return s + r.reshape(n, U, N_d)


def fdcnn_paper_forward(s: np.ndarray, params: np.ndarray, N_d: int, n_conv: int = 2) -> np.ndarray:
    """The paper's own FD-CNN (NEXT f2): per (symbol n, UE u), L_U = 1:
      * S x S matrix of the N_d symbols, S = ceil(sqrt(N_d)), contiguous row-major order, zero
        padding (P:170 and footnote); Re and Im matrices as 2 channels;
      * N^Conv 3x3 kernels, stride K_S = 1, zero padding keeping S x S, with bias;
      * element-wise ReLU, flatten to n_conv S^2 in (kernel, row, column) order;
      * fully connected linear output layer with 2 N_d neurons, with bias; neurons
        0..N_d-1 are the real parts and N_d..2N_d-1 the imaginary parts of s_tilde (reading P1).
    params: W1[n_conv][2][3][3], b1[n_conv], W2[2 N_d][n_conv S^2], b2[2 N_d]."""
    s = np.asarray(s, dtype=np.complex128)
    n, U, nd = s.shape
    assert nd == N_d
    S = int(np.ceil(np.sqrt(N_d)))
    p = np.asarray(params, dtype=np.float64)
    K = n_conv * S * S
    o = 0
    W1 = p[o:o + n_conv * 18].reshape(n_conv, 2, 3, 3); o += n_conv * 18
    b1 = p[o:o + n_conv]; o += n_conv
    W2 = p[o:o + 2 * N_d * K].reshape(2 * N_d, K); o += 2 * N_d * K
    b2 = p[o:o + 2 * N_d]; o += 2 * N_d
    assert o == p.size
    flat = np.zeros((n * U, S * S), dtype=np.complex128)
    flat[:, :N_d] = s.reshape(n * U, N_d)
    img = flat.reshape(n * U, S, S)
    h = np.stack([img.real, img.imag], axis=1)                      # [img][2][S][S]
    hp = np.zeros((h.shape[0], 2, S + 2, S + 2))
    hp[:, :, 1:S + 1, 1:S + 1] = h
    conv = np.broadcast_to(b1[None, :, None, None], (h.shape[0], n_conv, S, S)).copy()
    for dy in range(3):
        for dx in range(3):
            conv += np.einsum("oc,ncyx->noyx", W1[:, :, dy, dx], hp[:, :, dy:dy + S, dx:dx + S])
    feat = np.maximum(conv, 0.0).reshape(h.shape[0], K)            # ReLU, flatten
    out = feat @ W2.T + b2                                          # FC
    return (out[:, :N_d] + 1j * out[:, N_d:]).reshape(n, U, N_d)


def dpd_forward(cfg_head: str, s, params, chans, N_d, n_conv=2):
    """Dispatch on the FD-CNN variant: BASELINE residual stack (A1) or the paper head."""
    if cfg_head == "paper":
        return fdcnn_paper_forward(s, params, N_d, n_conv)
    return fdcnn_forward(s, params, chans, N_d)


# ============================================================================ channel / ZF
def channel_fd(h_taps: np.ndarray, N_ifft: int, N_d: int) -> np.ndarray:
    """H_hat_k = sum_t H_t exp(-j k 2 pi t / N) at the data bins (A9: unnormalised).
    h_taps [T][U][B] -> Hfd [N_d][U][B]."""
    h = np.asarray(h_taps, dtype=np.complex128)
    T = h.shape[0]
    k = data_bins(N_d, N_ifft)
    E = np.exp(-2j * np.pi * np.outer(k, np.arange(T)) / N_ifft)   # [N_d][T]
    return np.einsum("jt,tub->jub", E, h)


def zf_precoder(Hfd: np.ndarray, N_ifft: int, rho: float):
    """Zero-forcing precoder P_hat_k = alpha H^H (H H^H)^-1 (Eq. 6).

    alpha (reading A12): one scalar per channel realization so that, with
    E[s s^H] = I, the mean over antennas and TD samples of |x|^2 equals rho^2:
    by Parseval (unitary Eq. 2) sum_{b,m}|x|^2 = sum_j ||P_j s_j||^2, whose
    expectation is alpha^2 sum_j ||P0_j||_F^2 = alpha^2 sum_j tr(G_j^-1), so
    alpha = rho * sqrt(B N / sum_j tr(G_j^-1)).
    Returns P [N_d][B][U] (alpha folded in), alpha, P0 (unscaled)."""
    H = np.asarray(Hfd, dtype=np.complex128)
    B = H.shape[2]
    Hh = np.conj(np.transpose(H, (0, 2, 1)))                       # [N_d][B][U]
    G = H @ Hh                                                     # [N_d][U][U]
    Ginv = np.linalg.inv(G)
    P0 = Hh @ Ginv
    tr = np.real(np.trace(Ginv, axis1=1, axis2=2)).sum()
    alpha = rho * np.sqrt(B * N_ifft / tr)
    return alpha * P0, alpha, P0


# ============================================================================ precode / IDFT
def precode(P: np.ndarray, s_tilde: np.ndarray) -> np.ndarray:
    """x_hat_k = P_hat_k s_hat_k (Eq. 1).  P [N_d][B][U], s [n][U][N_d] -> X [n][B][N_d]."""
    return np.einsum("jbu,nuj->nbj", np.asarray(P, np.complex128), np.asarray(s_tilde, np.complex128))


def ofdm_modulate(X: np.ndarray, N_ifft: int) -> np.ndarray:
    """x_n = N^-1/2 sum_k x_hat_k exp(+j k 2 pi n / N) (Eq. 2), guards zero.
    X [n][B][N_d] -> x [n][B][N_ifft].  The FFT routine is the library primitive; it is
    pinned to the brute-force sum in tests."""
    X = np.asarray(X, dtype=np.complex128)
    full = np.zeros(X.shape[:-1] + (N_ifft,), dtype=np.complex128)
    full[..., data_bins(X.shape[-1], N_ifft)] = X
    return np.fft.ifft(full, axis=-1, norm="ortho")


# ============================================================================ GMP PA
def gmp_split(coef: np.ndarray, orders, L: int, M: int):
    """Unflatten SURVEY §8(b) order: a[p][l]; b[p>=3][l][g]; c[p>=3][l][g]."""
    Kp = len(orders)
    coef = np.asarray(coef, dtype=np.complex128)
    na = Kp * (L + 1)
    nb = (Kp - 1) * (L + 1) * M
    assert coef.shape[-1] == na + 2 * nb
    a = coef[..., :na].reshape(coef.shape[:-1] + (Kp, L + 1))
    b = coef[..., na:na + nb].reshape(coef.shape[:-1] + (Kp - 1, L + 1, M))
    c = coef[..., na + nb:].reshape(coef.shape[:-1] + (Kp - 1, L + 1, M))
    return a, b, c


def gmp_pa(x: np.ndarray, coef: np.ndarray, orders, L: int, M: int) -> np.ndarray:
    """GMP PA, Eq. (9) used as the PA model f_b (Eq. 7).

    With odd orders p (|u|^(p-1), reading A13), memory l = 0..L, cross-term lag g = 1..M:
      y_n = sum_p sum_l a_{p,l} u_{n-l} |u_{n-l}|^(p-1)
          + sum_{p>=3} sum_l sum_g ( b_{p,l,g} u_{n-l} |u_{n-l-g}|^(p-1)
                                   + c_{p,l,g} u_{n-l} |u_{n-l+g}|^(p-1) )
    Indices are circular within the OFDM symbol (A13).
    x [n][B][N], coef [B][n_coef] -> y [n][B][N]."""
    u = np.asarray(x, dtype=np.complex128)
    a, b, c = gmp_split(coef, orders, L, M)                  # a [B][Kp][L+1] ...
    y = np.zeros_like(u)

    def sh(v, d):                                            # sh(v, d)[n] = v[n - d] (circular)
        return np.roll(v, d, axis=-1)

    for ip, p in enumerate(orders):
        for l in range(L + 1):
            ul = sh(u, l)
            y += a[None, :, ip, l, None] * ul * np.abs(ul) ** (p - 1)
    for ip, p in enumerate(orders[1:]):
        for l in range(L + 1):
            ul = sh(u, l)
            for g in range(1, M + 1):
                y += b[None, :, ip, l, g - 1, None] * ul * np.abs(sh(u, l + g)) ** (p - 1)
                y += c[None, :, ip, l, g - 1, None] * ul * np.abs(sh(u, l - g)) ** (p - 1)
    return y


# ============================================================================ receive / SER
def channel_td(y: np.ndarray, h_taps: np.ndarray) -> np.ndarray:
    """Eq. (3), noiseless, circular (ideal cyclic prefix, A10):
    r_n = sum_t H_t y_{n-t}.  y [n][B][N], h [T][U][B] -> r [n][U][N]."""
    h = np.asarray(h_taps, dtype=np.complex128)
    y = np.asarray(y, dtype=np.complex128)
    r = np.zeros((y.shape[0], h.shape[1], y.shape[2]), dtype=np.complex128)
    for t in range(h.shape[0]):
        r += np.einsum("ub,nbm->num", h[t], np.roll(y, t, axis=-1))
    return r


def ue_receive(y: np.ndarray, Hfd: np.ndarray, N_d: int) -> np.ndarray:
    """y_hat_k = H_hat_k x^PA_k (Eq. 4-5, noiseless, A11), with x^PA_k the unitary
    DFT of the PA output at data bin k_j (A9).  y [n][B][N], Hfd [N_d][U][B] -> yhat [n][U][N_d]."""
    y = np.asarray(y, dtype=np.complex128)
    N = y.shape[-1]
    XPA = np.fft.fft(y, axis=-1, norm="ortho")[..., data_bins(N_d, N)]   # [n][B][N_d]
    return np.einsum("jub,nbj->nuj", np.asarray(Hfd, np.complex128), XPA)


def slice_ser(yhat: np.ndarray, alpha: float, idx: np.ndarray, M_qam: int, eps: float = 1e-4):
    """Nearest-point QAM decision on z = y_hat / alpha (genie alpha, A17) and the SER
    count against the transmitted indices (A18, A20).

    Per axis in level units v = z / c: d = clip(2 floor(v/2) + 1, -(m-1), m-1) (nearest odd
    level, ties upward).  'near' marks samples within eps (unit-energy units) of an interior
    decision boundary (the north star's decision-parity exclusion).
    Returns dec [n][U][N_d] (uint16), counts int64[3] = (errors, total, near)."""
    m = int(round(np.sqrt(M_qam)))
    c = 1.0 / np.sqrt(2.0 * (M_qam - 1) / 3.0)
    z = np.asarray(yhat, dtype=np.complex128) / alpha
    dec_axes, near = [], np.zeros(z.shape, dtype=bool)
    for v in (z.real / c, z.imag / c):
        d = np.clip(2.0 * np.floor(v / 2.0) + 1.0, -(m - 1), m - 1)
        dec_axes.append(((d + (m - 1)) / 2).astype(np.int64))
        bnd = 2.0 * np.round(v / 2.0)
        near |= (np.abs(v - bnd) < eps / c) & (np.abs(bnd) <= m - 2)
    dec = dec_axes[0] + m * dec_axes[1]
    err = int(np.count_nonzero(dec != np.asarray(idx, dtype=np.int64)))
    counts = np.array([err, dec.size, int(near.sum())], dtype=np.int64)
    return dec.astype(np.uint16), counts


# ============================================================================ impairments (NEXT f3)
# Counter-based RNG: Philox4x32-10 (Salmon, Moraes, Dror, Shaw, SC'11).  The GPU implements the
# same generator, so the noise of any (symbol, antenna/UE, sample) is reproducible anywhere.
PHILOX_M = (0xD2511F53, 0xCD9E8D57)
PHILOX_W = (0x9E3779B9, 0xBB67AE85)
STREAM_PA_NOISE, STREAM_AWGN = 1, 2


def philox4x32_10(ctr, key):
    """ctr uint32 [..., 4], key (k0, k1) -> uint32 [..., 4]; 10 rounds, key bumped between rounds."""
    mask = np.uint64(0xFFFFFFFF)
    c = [np.asarray(ctr)[..., i].astype(np.uint64) for i in range(4)]
    k0, k1 = np.uint64(key[0]), np.uint64(key[1])
    for _ in range(10):
        p0 = np.uint64(PHILOX_M[0]) * c[0]
        p1 = np.uint64(PHILOX_M[1]) * c[2]
        c = [(p1 >> np.uint64(32)) ^ c[1] ^ k0, p1 & mask, (p0 >> np.uint64(32)) ^ c[3] ^ k1, p0 & mask]
        k0 = (k0 + np.uint64(PHILOX_W[0])) & mask
        k1 = (k1 + np.uint64(PHILOX_W[1])) & mask
    return np.stack(c, axis=-1).astype(np.uint32)


def complex_gaussian(idx, stream, key64, std):
    """CN(0, std^2) noise for global sample indices idx: Philox counter (idx lo, idx hi, stream, 0),
    key (key64 lo, key64 hi); Box-Muller on the first two words, u = (x + 1/2) 2^-32."""
    idx = np.asarray(idx, dtype=np.uint64)
    ctr = np.stack([idx & np.uint64(0xFFFFFFFF), idx >> np.uint64(32),
                    np.full(idx.shape, stream, np.uint64), np.zeros(idx.shape, np.uint64)], axis=-1)
    x = philox4x32_10(ctr, (key64 & 0xFFFFFFFF, key64 >> 32)).astype(np.float64)
    u1 = (x[..., 0] + 0.5) * 2.0 ** -32
    u2 = (x[..., 1] + 0.5) * 2.0 ** -32
    r = np.sqrt(-2.0 * np.log(u1))
    return (std / np.sqrt(2.0)) * r * (np.cos(2 * np.pi * u2) + 1j * np.sin(2 * np.pi * u2))


def pa_impair(y, clip, noise_std, key64, symbols, B_total, b0=0):
    """PA saturation then measurement noise (order as SPEC pa_forward S:214): |y| > clip is
    scaled to clip with the phase kept; then + CN(0, noise_std^2) with the global sample index
    ((symbol * B_total + b0 + b) * N + m)."""
    y = np.asarray(y, dtype=np.complex128).copy()
    if clip > 0:
        a = np.abs(y)
        y = np.where(a > clip, y * (clip / np.maximum(a, 1e-300)), y)
    if noise_std > 0:
        n, Bl, N = y.shape
        sym = np.asarray(symbols, dtype=np.uint64)[:, None, None]
        b = np.arange(Bl, dtype=np.uint64)[None, :, None] + np.uint64(b0)
        m = np.arange(N, dtype=np.uint64)[None, None, :]
        y = y + complex_gaussian((sym * np.uint64(B_total) + b) * np.uint64(N) + m, STREAM_PA_NOISE, key64, noise_std)
    return y


def ue_awgn(yhat, n0, key64, symbols):
    """AWGN at the UEs: w_n ~ CN(0, N_0 I) per TD sample; under the unitary DFT (A9) its
    data-subcarrier image is CN(0, N_0) i.i.d., drawn here per global index ((symbol U + u) N_d + j)."""
    yhat = np.asarray(yhat, dtype=np.complex128)
    if n0 <= 0:
        return yhat
    n, U, Nd = yhat.shape
    sym = np.asarray(symbols, dtype=np.uint64)[:, None, None]
    u = np.arange(U, dtype=np.uint64)[None, :, None]
    j = np.arange(Nd, dtype=np.uint64)[None, None, :]
    return yhat + complex_gaussian((sym * np.uint64(U) + u) * np.uint64(Nd) + j, STREAM_AWGN, key64, np.sqrt(n0))


def csi_estimate(h_taps, h_err, eta):
    """H_t^est = sqrt(1 - eta) H_t + sqrt(eta) H_t^err."""
    return np.sqrt(1.0 - eta) * np.asarray(h_taps, np.complex128) + np.sqrt(eta) * np.asarray(h_err, np.complex128)


# ============================================================================ composition
def run_chain(s, idx, h_taps, coef, params, *, chans, orders, L, M, N_ifft, M_qam, rho=0.3, head="residual",
              n_conv=2, clip=0.0, pa_noise_std=0.0, awgn_n0=0.0, csi_eta=0.0, h_err=None, noise_key=0,
              symbols=None):
    """The whole hot path, stage by stage, optionally with the impairments
    of NEXT f3 (PA clip + measurement noise, AWGN, imperfect CSI).  Returns every stage output."""
    s = np.asarray(s, dtype=np.complex128)
    N_d = s.shape[-1]
    B = np.asarray(h_taps).shape[2]
    symbols = np.arange(s.shape[0]) if symbols is None else np.asarray(symbols)
    out = {}
    out["s_tilde"] = dpd_forward(head, s, params, chans, N_d, n_conv)
    out["Hfd"] = channel_fd(h_taps, N_ifft, N_d)
    Hest = out["Hfd"] if csi_eta <= 0 else channel_fd(csi_estimate(h_taps, h_err, csi_eta), N_ifft, N_d)
    out["P"], out["alpha"], _ = zf_precoder(Hest, N_ifft, rho)
    out["X"] = precode(out["P"], out["s_tilde"])
    out["x"] = ofdm_modulate(out["X"], N_ifft)
    out["y"] = gmp_pa(out["x"], coef, orders, L, M)
    if clip > 0 or pa_noise_std > 0:
        out["y"] = pa_impair(out["y"], clip, pa_noise_std, noise_key, symbols, B)
    out["yhat"] = ue_awgn(ue_receive(out["y"], out["Hfd"], N_d), awgn_n0, noise_key, symbols)
    out["dec"], out["counts"] = slice_ser(out["yhat"], out["alpha"], idx, M_qam)
    return out


def run_config_redraw(cfg, inp, h_taps_per_symbol):
    """Per-symbol channel redraw ("coherence time of one OFDM symbol"; NEXT f4): symbol n uses
    its own taps, hence its own Hfd_n, P_n and alpha_n (A12 per realisation).  Stage outputs are
    stacked over symbols; alpha is the per-symbol vector; counts are summed."""
    outs = []
    for i, n in enumerate(inp["symbols"]):
        sub = dict(inp)
        sub.update(s=inp["s"][i:i + 1], idx=inp["idx"][i:i + 1], symbols=np.array([n]),
                   h_taps=h_taps_per_symbol[i])
        outs.append(run_config(cfg, sub))
    res = {k: np.concatenate([o[k] for o in outs]) for k in ("s_tilde", "x", "y", "yhat", "dec")}
    res["P"] = np.stack([o["P"] for o in outs])
    res["Hfd"] = np.stack([o["Hfd"] for o in outs])
    res["alpha"] = np.array([o["alpha"] for o in outs])
    res["counts"] = np.sum([o["counts"] for o in outs], axis=0)
    return res


def run_config(cfg, inp):
    """run_chain with a workload.configs.ChainConfig and a workload.gen.make_inputs bundle.  The
    transmitted symbols are derived here from the QAM indices (qam_points), rounded to
    complex64 like the canonical GPU input (the oracle runs on the canonical fp32
    inputs upcast exactly), so the oracle does not take the generator's symbol values."""
    s = qam_points(inp["idx"], cfg.M_qam).astype(np.complex64).astype(np.complex128)
    return run_chain(s, inp["idx"], inp["h_taps"], inp["coef"], inp["params"],
                     chans=cfg.chans, orders=cfg.orders, L=cfg.L, M=cfg.M,
                     N_ifft=cfg.N_ifft, M_qam=cfg.M_qam, rho=cfg.rho, head=cfg.head, n_conv=cfg.n_conv,
                     clip=cfg.clip, pa_noise_std=cfg.pa_noise_std, awgn_n0=cfg.awgn_n0, csi_eta=cfg.csi_eta,
                     h_err=inp.get("h_err"), noise_key=inp.get("noise_key", 0), symbols=inp.get("symbols"))

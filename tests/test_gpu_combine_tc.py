"""GPU parity of the tensor-core channel sum (Eq. 5) with fused slicing / SER
through the C ABI (ue_combine, ue_combine_ser; fd_set_combine_path 2 = tensor cores for
9 <= U <= 32) against the fp64 oracle einsum + slicer: y_hat at 2e-5, decisions identical
outside the 1e-4 band element by element, SER counters equal to the decisions; the SIMT kernel
(fd_set_combine_path(1)) agrees to 2e-5; accumulate mode adds onto y_hat."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fdpd_oracle as O

pytestmark = pytest.mark.gpu
TOL = 2e-5


@pytest.fixture(scope="module")
def F():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2205_05158_b200 import fdpd
    fdpd.lib()
    yield fdpd
    fdpd.set_combine_path(0)


def rel(a, b):
    a = np.asarray(a, dtype=np.complex128)
    b = np.asarray(b, dtype=np.complex128)
    return float(np.linalg.norm((a - b).ravel()) / max(np.linalg.norm(b.ravel()), 1e-300))


def dev(x, dtype=torch.complex64):
    return torch.from_numpy(np.ascontiguousarray(x)).to("cuda", dtype)


def crandn(rng, *shape, scale=1.0):
    return (scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))).astype(np.complex64)


def near_mask(yhat, alpha, M, eps=1e-4):
    m = int(round(np.sqrt(M)))
    cst = 1.0 / np.sqrt(2.0 * (M - 1) / 3.0)
    z = np.asarray(yhat, np.complex128) / alpha
    near = np.zeros(z.shape, bool)
    for v in (z.real / cst, z.imag / cst):
        bnd = 2.0 * np.round(v / 2.0)
        near |= (np.abs(v - bnd) < eps / cst) & (np.abs(bnd) <= m - 2)
    return near


@pytest.mark.parametrize("n,B,U,Nd", [(32, 512, 32, 3300),    # C5 bench batch
                                      (128, 256, 16, 3300),   # C4 bench batch
                                      (37, 200, 12, 70),      # ragged symbols / antennas / users
                                      (5, 24, 24, 38),        # N_d % 4 != 0
                                      (64, 64, 32, 600),      # Mode A shard (64 antennas) at 2 symbol tiles
                                      (1, 17, 9, 36)])
def test_combine_ser_tc(F, n, B, U, Nd):
    rng = np.random.default_rng(n * 17 + B + U)
    M_qam = 256
    XPA = crandn(rng, n, B, Nd, scale=0.3)
    h = crandn(rng, U, B, Nd, scale=0.3)
    want = np.einsum("ubj,nbj->nuj", h.astype(np.complex128), XPA.astype(np.complex128))
    alpha = float(np.sqrt(np.mean(np.abs(want) ** 2)))                 # z at unit scale
    idx = rng.integers(0, M_qam, size=(n, U, Nd)).astype(np.uint16)
    d_idx = dev(idx.astype(np.int32), torch.int32).to(torch.uint16)
    F.set_combine_path(2)
    dec = torch.zeros((n, U, Nd), dtype=torch.uint16, device="cuda")
    yhat, counts, _ = F.ue_combine_ser(dev(XPA), dev(h), alpha, d_idx, M_qam, dec=dec)
    y = yhat.cpu().numpy()
    assert rel(y, want) < TOL
    dec_o, c_o = O.slice_ser(want, alpha, idx, M_qam)
    near = near_mask(want, alpha, M_qam)
    dg = dec.cpu().numpy()
    assert np.array_equal(dg[~near], dec_o[~near])
    c = counts.cpu().numpy()
    assert c[1] == n * U * Nd and c[0] == int((dg != idx).sum())
    # the SIMT kernel on the same inputs
    F.set_combine_path(1)
    y_simt = F.ue_combine(dev(XPA), dev(h)).cpu().numpy()
    F.set_combine_path(2)
    assert rel(y, y_simt) < TOL
    # ue_combine (no slicing) and accumulate
    y2 = F.ue_combine(dev(XPA), dev(h))
    assert torch.equal(y2, yhat)
    F.ue_combine(dev(XPA), dev(h), out=y2, accumulate=True)
    assert rel(y2.cpu().numpy(), 2 * want) < TOL

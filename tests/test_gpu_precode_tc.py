"""GPU parity of the tensor-core precode (Eq. 1; SURVEY §8(b) `math`) through the C ABI
against the fp64 oracle contraction O.precode:

  * FD_MATH_FP32_TC (split TF32, FP32-accurate) at the C4 / C5 shapes and batches the bench
    runs, and ragged antenna / symbol / subcarrier tiles: relative L2 <= 2e-5 (the FP32 bar);
  * FD_MATH_TF32 (one TF32 pass; BASELINE configs[2] "TF32 tensor-core precoding variant"):
    relative L2 <= 2e-3 at C3 with the bench batch;
  * the packed-precoder path (precode_pack + precode_packed) is bit-identical to the plain one,
    and precode_pack is exactly the documented relayout."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")

from oracle import fdpd_oracle as O
from workload import configs, gen

pytestmark = pytest.mark.gpu

TOL_FP32, TOL_TF32 = 2e-5, 2e-3


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


def crandn(rng, *shape, scale=1.0):
    return (scale * (rng.standard_normal(shape) + 1j * rng.standard_normal(shape))).astype(np.complex64)


def test_precode_pack_layout(F):
    rng = np.random.default_rng(0)
    B, U, Nd = 37, 12, 70
    P = crandn(rng, B, U, Nd)
    Ppk = F.precode_pack(dev(P)).cpu().numpy()
    want = np.concatenate([P.real.transpose(2, 0, 1), P.imag.transpose(2, 0, 1)], axis=2)   # [j][b][2U]
    assert Ppk.shape == (Nd, B, 2 * U)
    assert np.array_equal(Ppk, want.astype(np.float32))


@pytest.mark.parametrize("n,B,U,Nd", [(32, 512, 32, 3300),    # C5 shape, bench batch
                                      (128, 256, 16, 3300),   # C4 shape, bench batch
                                      (37, 200, 12, 70),      # ragged everything
                                      (1, 8, 4, 36),          # C1 shape
                                      (65, 64, 4, 600),       # C2 shape, ragged symbol tile
                                      (33, 130, 32, 38)])
def test_precode_fp32tc(F, n, B, U, Nd):
    rng = np.random.default_rng(n * 7 + B + U)
    P = crandn(rng, B, U, Nd)
    s = crandn(rng, n, U, Nd)
    want = O.precode(P.transpose(2, 0, 1), s)
    got = F.precode(dev(P), dev(s), math=F.MATH_FP32_TC)
    torch.cuda.synchronize()
    assert got.shape == (n, B, Nd)
    e = rel(got.cpu().numpy(), want)
    assert e < TOL_FP32, e
    got_pk = F.precode_packed(F.precode_pack(dev(P)), dev(s), math=F.MATH_FP32_TC)
    assert torch.equal(got_pk, got)                   # same arithmetic, same order: bit-identical


@pytest.mark.parametrize("n,B,U,Nd", [(512, 128, 8, 1200),    # C3, bench batch: the TF32 variant
                                      (70, 512, 32, 3300), (9, 37, 4, 70)])
def test_precode_tf32(F, n, B, U, Nd):
    rng = np.random.default_rng(n + B + U)
    P = crandn(rng, B, U, Nd)
    s = crandn(rng, n, U, Nd)
    want = O.precode(P.transpose(2, 0, 1), s)
    got = F.precode(dev(P), dev(s), math=F.MATH_TF32)
    e = rel(got.cpu().numpy(), want)
    assert 1e-6 < e < TOL_TF32, e                     # TF32 (10-bit mantissa): ~1e-3 class, not FP32
    got_pk = F.precode_packed(F.precode_pack(dev(P)), dev(s), math=F.MATH_TF32)
    assert torch.equal(got_pk, got)


def test_precode_tc_zf_precoder_c5(F):
    """The real ZF precoder of C5 (alpha folded in) on the 32-symbol bench batch of the
    generator's QAM symbols: X at 2e-5 (split TF32) and 2e-3 (TF32)."""
    cfg = configs.C5
    inp = gen.make_inputs(cfg, list(range(32)))
    h_fd, P, alpha = F.zf_precoder_build(dev(inp["h_taps"]), cfg.N_ifft, cfg.N_d, cfg.rho)
    s = dev(inp["s"])
    Pn = P.cpu().numpy()
    want = O.precode(Pn.transpose(2, 0, 1), inp["s"])
    Ppk = F.precode_pack(P)
    assert rel(F.precode_packed(Ppk, s, math=F.MATH_FP32_TC).cpu().numpy(), want) < TOL_FP32
    assert rel(F.precode_packed(Ppk, s, math=F.MATH_TF32).cpu().numpy(), want) < TOL_TF32


def test_precode_tc_errors(F):
    P = torch.zeros((8, 6, 36), dtype=torch.complex64, device="cuda")
    s = torch.zeros((2, 6, 36), dtype=torch.complex64, device="cuda")
    with pytest.raises(F.FdpdError):
        F.precode(P, s, math=F.MATH_TF32)             # U % 4 != 0
    with pytest.raises(F.FdpdError):
        F.precode(P, s, math=7)
    P = torch.zeros((8, 36, 36), dtype=torch.complex64, device="cuda")
    s = torch.zeros((2, 36, 36), dtype=torch.complex64, device="cuda")
    with pytest.raises(F.FdpdError):
        F.precode(P, s, math=F.MATH_FP32_TC)          # U > 32
    empty = F.precode(P[:, :32].contiguous(), s[:0, :32].contiguous(), math=F.MATH_FP32_TC)
    assert empty.shape == (0, 8, 36)

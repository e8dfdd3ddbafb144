"""Thin ctypes binding of libfdpd.so (include/fdpd.h) — argument marshalling only.

Each function has the C entry point's name, takes CUDA torch tensors, allocates
outputs with torch when ``out`` is not given (device memory plumbing), passes raw
pointers plus the current torch stream, and raises ``FdpdError`` on a non-OK
status.  Every step of the path runs in libfdpd's kernels; there is no CPU path.
"""
from __future__ import annotations

import ctypes as C
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# FDPD_LIB: an alternative build of the same library (tools/ A/B experiments of compile-time variants)
LIB_PATH = os.environ.get("FDPD_LIB") or os.path.join(_HERE, "libfdpd.so")

FD_OK, FD_ERR_ARG, FD_ERR_NUMERIC, FD_ERR_CUDA = 0, 2, 3, 4

_vp, _i, _ll, _f, _sz = C.c_void_p, C.c_int, C.c_longlong, C.c_float, C.c_size_t
_ip = C.POINTER(C.c_int)

FD_CHAIN_MAX_LAYERS = 8


class ChainDesc(C.Structure):
    """fd_chain_desc (include/fdpd.h)."""
    _fields_ = [("U", C.c_int), ("B", C.c_int), ("T", C.c_int), ("N_d", C.c_int), ("N_ifft", C.c_int),
                ("M_qam", C.c_int), ("n_layers", C.c_int), ("chans", C.c_int * (FD_CHAIN_MAX_LAYERS + 1)),
                ("n_orders", C.c_int), ("orders", C.c_int * 8), ("L", C.c_int), ("M", C.c_int),
                ("rho", C.c_float), ("boundary_eps", C.c_float), ("head", C.c_int), ("n_conv", C.c_int)]


_cp = C.POINTER(C.c_void_p)


class Impairments(C.Structure):
    """fd_impair (include/fdpd.h): PA clip + measurement noise, AWGN, imperfect CSI (NEXT f3)."""
    _fields_ = [("clip", C.c_float), ("pa_noise_std", C.c_float), ("awgn_n0", C.c_float), ("csi_eta", C.c_float),
                ("noise_key", C.c_ulonglong), ("sym0", C.c_longlong), ("b0", C.c_int), ("B_total", C.c_int)]


_imp = C.POINTER(Impairments)

# name -> (restype, argtypes), mirroring include/fdpd.h
SIGNATURES = {
    "fd_last_error": (C.c_char_p, []),
    "fd_version": (_i, []),
    "fd_shutdown": (None, []),
    "fd_set_cnn_path": (_i, [_i]),
    "fd_set_cnn_tc_precision": (_i, [_i]),
    "fd_set_chain_split": (_i, [_i]),
    "fd_set_gmp_path": (_i, [_i]),
    "fd_debug_poison_smem": (_i, [C.c_uint, _vp]),
    "fd_set_combine_path": (_i, [_i]),
    "fdcnn_workspace_bytes": (_sz, [_ip, _i, _ll, _i, _i]),
    "fdcnn_forward": (_i, [_vp, _ip, _i, _vp, _vp, _vp, _sz, _ll, _i, _i, _vp]),
    "fdcnn_paper_workspace_bytes": (_sz, [_i, _ll, _i, _i]),
    "fdcnn_paper_forward": (_i, [_vp, _i, _vp, _vp, _vp, _sz, _ll, _i, _i, _vp]),
    "zf_workspace_bytes": (_sz, [_i]),
    "zf_precoder_build": (_i, [_vp, _i, _i, _i, _i, _i, _f, _i, _i, _vp, _vp, C.POINTER(C.c_float), _vp, _sz, _vp]),
    "precode": (_i, [_vp, _vp, _vp, _ll, _i, _i, _i, _i, _vp]),
    "precode_pack_bytes": (_sz, [_i, _i, _i]),
    "precode_pack": (_i, [_vp, _vp, _i, _i, _i, _vp]),
    "precode_packed": (_i, [_vp, _vp, _vp, _ll, _i, _i, _i, _i, _vp]),
    "ofdm_modulate": (_i, [_vp, _vp, _ll, _i, _i, _i, _vp]),
    "gmp_pa": (_i, [_vp, _vp, _vp, _ip, _i, _i, _i, _ll, _i, _i, _vp]),
    "chain_tx": (_i, [_vp, _vp, _vp, _vp, _ip, _i, _i, _i, _ll, _i, _i, _i, _i, _vp]),
    "chain_txrx": (_i, [_vp, _vp, _vp, _vp, _vp, _ip, _i, _i, _i, _ll, _i, _i, _i, _i, _vp]),
    "ue_combine": (_i, [_vp, _vp, _vp, _ll, _i, _i, _i, _i, _vp]),
    "ue_combine_ser": (_i, [_vp, _vp, _vp, _f, _vp, _i, _vp, _vp, _ll, _i, _i, _i, _f, _vp]),
    "ue_combine_peer": (_i, [_vp, _vp, C.POINTER(C.c_void_p), _i, _i, _ll, _i, _i, _i, _vp]),
    "ue_reduce_ser": (_i, [_vp, _i, _vp, _f, _vp, _i, _vp, _vp, _ll, _i, _i, _f, _vp]),
    "ue_receive_workspace_bytes": (_sz, [_ll, _i, _i]),
    "ue_receive": (_i, [_vp, _vp, _vp, _vp, _sz, _ll, _i, _i, _i, _i, _i, _vp]),
    "ue_slice_ser": (_i, [_vp, _f, _vp, _i, _vp, _vp, _ll, _i, _i, _f, _vp]),
    "ue_receive_ser": (_i, [_vp, _vp, _vp, _vp, _sz, _f, _vp, _i, _vp, _vp, _ll, _i, _i, _i, _i, _f, _vp]),
    "chain_txrx_ex": (_i, [_vp, _vp, _vp, _vp, _vp, _ip, _i, _i, _i, _ll, _i, _i, _i, _i, _imp, _vp]),
    "chain_txrx_pre": (_i, [_vp, _vp, _vp, _vp, _ip, _i, _i, _i, _ll, _i, _i, _i, _imp, _vp]),
    "zf_precoder_build_ex": (_i, [_vp, _vp, _f, _i, _i, _i, _i, _i, _f, _i, _i, _vp, _vp, C.POINTER(C.c_float), _vp,
                                  _sz, _vp]),
    "ue_combine_ser_ex": (_i, [_vp, _vp, _vp, _f, _vp, _i, _vp, _vp, _ll, _i, _i, _i, _f, _imp, _vp]),
    "zf_batched_workspace_bytes": (_sz, [_i, _i]),
    "zf_precoder_build_batched": (_i, [_vp, _i, _i, _i, _i, _i, _i, _f, _i, _i, _vp, _vp, _vp, _vp, _vp, _sz, _vp]),
    "chain_txrx_ps": (_i, [_vp, _vp, _vp, _vp, _vp, _ip, _i, _i, _i, _ll, _i, _i, _i, _i, _imp, _vp]),
    "ue_combine_ser_ps": (_i, [_vp, _vp, _vp, _vp, _vp, _i, _vp, _vp, _ll, _i, _i, _i, _f, _imp, _vp]),
    "fd_chain_create": (_i, [_cp, C.POINTER(ChainDesc), _vp, _vp, _vp, _ll, _vp]),
    "fd_chain_alpha": (_f, [_vp]),
    "fd_chain_destroy": (None, [_vp]),
    "fd_chain_run_device": (_i, [_vp, _vp, _vp, _ll, _vp, _vp, _vp]),
    "fd_chain_run_host": (_i, [_vp, _vp, _vp, _ll, _vp, _vp]),
    "fd_chain_run_host_qam": (_i, [_vp, _vp, _ll, _vp, _vp]),
    "qam_map": (_i, [_vp, _vp, _ll, _i, _vp]),
}


class FdpdError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"libfdpd status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load libfdpd.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with `python -m paper_2205_05158_b200.build` "
                               "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def _check(status: int):
    if status != FD_OK:
        raise FdpdError(status, lib().fd_last_error().decode())


def _ints(vals):
    arr = (C.c_int * len(vals))(*[int(v) for v in vals])
    return arr


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _dev(t, dtype, name):
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (there is no CPU path)")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _stream(t):
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _ws(nbytes, like):
    return torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=like.device)


# ----------------------------------------------------------------------------- a1
CNN_AUTO, CNN_SIMT, CNN_TENSOR = 0, 1, 2
# FD_SPLIT_PRECODE_MIN_U of include/fdpd.h: from this many users the chain runs precode ->
# chain_txrx_pre instead of the fused-prologue chain_txrx (same policy as the native runtime)
SPLIT_PRECODE_MIN_U = 16


def set_combine_path(mode: int):
    """0 = auto (the FP32 SIMT kernels), 1 = FP32 SIMT, 2 = tensor cores for 9 <= U <= 32."""
    _check(lib().fd_set_combine_path(int(mode)))


def set_cnn_tc_precision(mode: int):
    """0 = FP16 split (default), 1 = TF32 split for the tensor-core hidden layers."""
    _check(lib().fd_set_cnn_tc_precision(int(mode)))


def set_cnn_path(path: int):
    """Choose the FD-CNN implementation (include/fdpd.h fd_set_cnn_path): CNN_AUTO (tensor
    cores where every hidden width is 16/32/64), CNN_SIMT or CNN_TENSOR.  Process-wide."""
    _check(lib().fd_set_cnn_path(int(path)))


def qam_map(idx, M_qam, out=None):
    """a0: complex64 QAM points of uint16 indices on the device (include/fdpd.h qam_map)."""
    _dev(idx, torch.uint16, "idx")
    out = torch.empty(idx.shape, dtype=torch.complex64, device=idx.device) if out is None else out
    _check(lib().qam_map(_ptr(idx), _ptr(out), idx.numel(), int(M_qam), _stream(idx)))
    return out


def set_gmp_path(mode: int):
    """GMP of the N = 16384 cluster chain (include/fdpd.h fd_set_gmp_path): 0 = auto (= FP32 SIMT), 1 = FP32 SIMT,
    2 = tensor cores (C4 / C5 GMP shape).  Process-wide."""
    _check(lib().fd_set_gmp_path(int(mode)))


def debug_poison_smem(pattern: int):
    """Test support (include/fdpd.h fd_debug_poison_smem): shared memory of every SM := pattern."""
    _check(lib().fd_debug_poison_smem(int(pattern) & 0xFFFFFFFF,
                                      C.c_void_p(torch.cuda.current_stream().cuda_stream)))


def set_chain_split(mode: int):
    """Cluster split of the N = 8192 / 16384 chain kernels (include/fdpd.h fd_set_chain_split):
    0 = auto (default), 1 = never.  Process-wide."""
    _check(lib().fd_set_chain_split(int(mode)))


def fdcnn_forward(params, chans, s_in, out=None, workspace=None):
    """s_tilde = s + CNN(s)  (include/fdpd.h fdcnn_forward).  s_in complex64 [n_sym][U][N_d]."""
    _dev(params, torch.float32, "params")
    _dev(s_in, torch.complex64, "s_in")
    n_sym, U, N_d = s_in.shape
    ch = _ints(chans)
    nl = len(chans) - 1
    out = torch.empty_like(s_in) if out is None else _dev(out, torch.complex64, "out")
    need = lib().fdcnn_workspace_bytes(ch, nl, n_sym, U, N_d)
    if workspace is None or workspace.numel() < need:
        workspace = _ws(need, s_in)
    _check(lib().fdcnn_forward(_ptr(params), ch, nl, _ptr(s_in), _ptr(out), _ptr(workspace), workspace.numel(),
                               n_sym, U, N_d, _stream(s_in)))
    return out


def fdcnn_paper_forward(params, n_conv, s_in, out=None, workspace=None):
    """Paper FD-CNN head (include/fdpd.h fdcnn_paper_forward).  s_in complex64 [n_sym][U][N_d]."""
    _dev(params, torch.float32, "params")
    _dev(s_in, torch.complex64, "s_in")
    n_sym, U, N_d = s_in.shape
    out = torch.empty_like(s_in) if out is None else _dev(out, torch.complex64, "out")
    need = lib().fdcnn_paper_workspace_bytes(n_conv, n_sym, U, N_d)
    if workspace is None or workspace.numel() < need:
        workspace = _ws(need, s_in)
    _check(lib().fdcnn_paper_forward(_ptr(params), n_conv, _ptr(s_in), _ptr(out), _ptr(workspace),
                                     workspace.numel(), n_sym, U, N_d, _stream(s_in)))
    return out


# ----------------------------------------------------------------------------- a2
def zf_precoder_build(h_taps, N_ifft, N_d, rho, b0=0, B_loc=None):
    """Returns (h_fd [U][B_loc][N_d], P [B_loc][U][N_d], alpha) — include/fdpd.h zf_precoder_build."""
    _dev(h_taps, torch.complex64, "h_taps")
    T, U, B = h_taps.shape
    B_loc = B - b0 if B_loc is None else B_loc
    h_fd = torch.empty((U, B_loc, N_d), dtype=torch.complex64, device=h_taps.device)
    P = torch.empty((B_loc, U, N_d), dtype=torch.complex64, device=h_taps.device)
    ws = _ws(lib().zf_workspace_bytes(N_d), h_taps)
    a = C.c_float(0.0)
    _check(lib().zf_precoder_build(_ptr(h_taps), T, U, B, N_ifft, N_d, float(rho), b0, B_loc, _ptr(h_fd), _ptr(P),
                                   C.byref(a), _ptr(ws), ws.numel(), _stream(h_taps)))
    return h_fd, P, float(a.value)


def zf_precoder_build_ex(h_taps, h_err, eta, N_ifft, N_d, rho, b0=0, B_loc=None):
    """zf_precoder_build with imperfect CSI: precoder from sqrt(1-eta) H + sqrt(eta) H_err."""
    _dev(h_taps, torch.complex64, "h_taps")
    _dev(h_err, torch.complex64, "h_err")
    T, U, B = h_taps.shape
    B_loc = B - b0 if B_loc is None else B_loc
    h_fd = torch.empty((U, B_loc, N_d), dtype=torch.complex64, device=h_taps.device)
    P = torch.empty((B_loc, U, N_d), dtype=torch.complex64, device=h_taps.device)
    ws = _ws(lib().zf_workspace_bytes(N_d), h_taps)
    a = C.c_float(0.0)
    _check(lib().zf_precoder_build_ex(_ptr(h_taps), _ptr(h_err), float(eta), T, U, B, N_ifft, N_d, float(rho), b0,
                                      B_loc, _ptr(h_fd), _ptr(P), C.byref(a), _ptr(ws), ws.numel(),
                                      _stream(h_taps)))
    return h_fd, P, float(a.value)


def zf_precoder_build_batched(h_taps_all, N_ifft, N_d, rho, out=None):
    """Per-symbol channel redraw (NEXT f4): h_taps_all [n_ch][T][U][B] -> (h_fd_all, P_all,
    alpha_dev [n_ch] float32 on the device, status int32 [1] on the device); asynchronous."""
    _dev(h_taps_all, torch.complex64, "h_taps_all")
    n_ch, T, U, B = h_taps_all.shape
    dv = h_taps_all.device
    if out is None:
        out = (torch.empty((n_ch, U, B, N_d), dtype=torch.complex64, device=dv),
               torch.empty((n_ch, B, U, N_d), dtype=torch.complex64, device=dv),
               torch.empty(n_ch, dtype=torch.float32, device=dv),
               torch.zeros(1, dtype=torch.int32, device=dv),
               _ws(lib().zf_batched_workspace_bytes(n_ch, N_d), h_taps_all))
    h_fd, P, alpha, status, ws = out
    _check(lib().zf_precoder_build_batched(_ptr(h_taps_all), n_ch, T, U, B, N_ifft, N_d, float(rho), 0, B,
                                           _ptr(h_fd), _ptr(P), _ptr(alpha), _ptr(status), _ptr(ws), ws.numel(),
                                           _stream(h_taps_all)))
    return out


def chain_txrx_pre(X, coef, orders, L, M, N_ifft, imp=None, y=None, XPA=None):
    """chain_txrx on a precoded spectrum X [n_sym][B_loc][N_d] (output of precode)."""
    _dev(X, torch.complex64, "X")
    _dev(coef, torch.complex64, "coef")
    n_sym, B, N_d = X.shape
    if y is None:
        y = torch.empty((n_sym, B, N_ifft), dtype=torch.complex64, device=X.device)
    if XPA is None:
        XPA = torch.empty((n_sym, B, N_d), dtype=torch.complex64, device=X.device)
    _check(lib().chain_txrx_pre(_ptr(X), _ptr(coef), _ptr(y), _ptr(XPA), _ints(orders), len(orders), L, M, n_sym, B,
                                N_d, N_ifft, C.byref(imp) if imp else None, _stream(X)))
    return y, XPA


def chain_txrx_ps(P_all, s_tilde, coef, orders, L, M, N_ifft, imp=None, y=None, XPA=None):
    """chain_txrx with per-symbol precoders P_all [n_sym][B_loc][U][N_d]."""
    _dev(P_all, torch.complex64, "P_all")
    _dev(s_tilde, torch.complex64, "s_tilde")
    _dev(coef, torch.complex64, "coef")
    n_sym, B, U, N_d = P_all.shape
    if y is None:
        y = torch.empty((n_sym, B, N_ifft), dtype=torch.complex64, device=P_all.device)
    if XPA is None:
        XPA = torch.empty((n_sym, B, N_d), dtype=torch.complex64, device=P_all.device)
    _check(lib().chain_txrx_ps(_ptr(P_all), _ptr(s_tilde), _ptr(coef), _ptr(y), _ptr(XPA), _ints(orders),
                               len(orders), L, M, n_sym, B, U, N_d, N_ifft, C.byref(imp) if imp else None,
                               _stream(P_all)))
    return y, XPA


def ue_combine_ser_ps(XPA, h_fd_all, alpha_dev, tx_idx, M_qam, imp=None, yhat=None, counts=None, dec=None,
                      boundary_eps=1e-4):
    _dev(XPA, torch.complex64, "XPA")
    _dev(h_fd_all, torch.complex64, "h_fd_all")
    _dev(alpha_dev, torch.float32, "alpha_dev")
    _dev(tx_idx, torch.uint16, "tx_idx")
    n_sym, B, N_d = XPA.shape
    U = h_fd_all.shape[1]
    if yhat is None:
        yhat = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=XPA.device)
    if counts is None:
        counts = torch.zeros(3, dtype=torch.int64, device=XPA.device)
    _check(lib().ue_combine_ser_ps(_ptr(XPA), _ptr(h_fd_all), _ptr(yhat), _ptr(alpha_dev), _ptr(tx_idx), M_qam,
                                   _ptr(dec), _ptr(counts), n_sym, B, U, N_d, float(boundary_eps),
                                   C.byref(imp) if imp else None, _stream(XPA)))
    return yhat, counts, dec


def make_impairments(clip=0.0, pa_noise_std=0.0, awgn_n0=0.0, csi_eta=0.0, noise_key=0, sym0=0, b0=0, B_total=0):
    return Impairments(float(clip), float(pa_noise_std), float(awgn_n0), float(csi_eta), int(noise_key), int(sym0),
                       int(b0), int(B_total))


# ----------------------------------------------------------------------------- a3-a5
MATH_FP32, MATH_TF32, MATH_FP32_TC = 0, 1, 2
MATH = {"simt": MATH_FP32, "fp32": MATH_FP32, "tf32": MATH_TF32, "fp32tc": MATH_FP32_TC}


def auto_precode_math(U: int) -> str:
    """The precode of the split path (U >= SPLIT_PRECODE_MIN_U): FP32-accurate tensor cores where
    they apply (U % 4 == 0, U <= 32; measured C5 0.47 vs 0.61 ms per 32 symbols), else FP32 SIMT —
    the same policy as the native runtime (fd_chain_create)."""
    return "fp32tc" if U >= SPLIT_PRECODE_MIN_U and U % 4 == 0 and U <= 32 else "simt"


def precode(P, s, out=None, math=MATH_FP32):
    """P [B][U][N_d], s [n][U][N_d] -> X [n][B][N_d]; math 0 FP32 SIMT, 1 TF32 / 2 split-TF32 tensor cores."""
    _dev(P, torch.complex64, "P")
    _dev(s, torch.complex64, "s")
    B, U, N_d = P.shape
    n_sym = s.shape[0]
    out = torch.empty((n_sym, B, N_d), dtype=torch.complex64, device=s.device) if out is None else out
    _check(lib().precode(_ptr(P), _ptr(s), _ptr(out), n_sym, B, U, N_d, int(math), _stream(s)))
    return out


def precode_pack(P, out=None):
    """P [B][U][N_d] complex64 -> Ppk [N_d][B][2U] float32 (per-subcarrier tensor-core layout)."""
    _dev(P, torch.complex64, "P")
    B, U, N_d = P.shape
    out = torch.empty((N_d, B, 2 * U), dtype=torch.float32, device=P.device) if out is None else out
    _check(lib().precode_pack(_ptr(P), _ptr(out), B, U, N_d, _stream(P)))
    return out


def precode_packed(Ppk, s, out=None, math=MATH_FP32_TC):
    _dev(Ppk, torch.float32, "Ppk")
    _dev(s, torch.complex64, "s")
    N_d, B, U2 = Ppk.shape
    n_sym = s.shape[0]
    out = torch.empty((n_sym, B, N_d), dtype=torch.complex64, device=s.device) if out is None else out
    _check(lib().precode_packed(_ptr(Ppk), _ptr(s), _ptr(out), n_sym, B, U2 // 2, N_d, int(math), _stream(s)))
    return out


def ofdm_modulate(X, N_ifft, out=None):
    _dev(X, torch.complex64, "X")
    n_sym, B, N_d = X.shape
    out = torch.empty((n_sym, B, N_ifft), dtype=torch.complex64, device=X.device) if out is None else out
    _check(lib().ofdm_modulate(_ptr(X), _ptr(out), n_sym, B, N_d, N_ifft, _stream(X)))
    return out


def gmp_pa(x, coef, orders, L, M, out=None):
    _dev(x, torch.complex64, "x")
    _dev(coef, torch.complex64, "coef")
    n_sym, B, N = x.shape
    out = torch.empty_like(x) if out is None else out
    _check(lib().gmp_pa(_ptr(x), _ptr(coef), _ptr(out), _ints(orders), len(orders), L, M, n_sym, B, N, _stream(x)))
    return out


def chain_tx(P, s_tilde, coef, orders, L, M, N_ifft, out=None):
    """Fused precode -> IDFT -> GMP: y [n_sym][B_loc][N_ifft]."""
    _dev(P, torch.complex64, "P")
    _dev(s_tilde, torch.complex64, "s_tilde")
    _dev(coef, torch.complex64, "coef")
    B, U, N_d = P.shape
    n_sym = s_tilde.shape[0]
    out = torch.empty((n_sym, B, N_ifft), dtype=torch.complex64, device=P.device) if out is None else out
    _check(lib().chain_tx(_ptr(P), _ptr(s_tilde), _ptr(coef), _ptr(out), _ints(orders), len(orders), L, M,
                          n_sym, B, U, N_d, N_ifft, _stream(P)))
    return out


def chain_txrx_ex(P, s_tilde, coef, orders, L, M, N_ifft, imp, y=None, XPA=None):
    """chain_txrx with PA clip + measurement noise (imp: Impairments)."""
    _dev(P, torch.complex64, "P")
    _dev(s_tilde, torch.complex64, "s_tilde")
    _dev(coef, torch.complex64, "coef")
    B, U, N_d = P.shape
    n_sym = s_tilde.shape[0]
    if y is None:
        y = torch.empty((n_sym, B, N_ifft), dtype=torch.complex64, device=P.device)
    if XPA is None:
        XPA = torch.empty((n_sym, B, N_d), dtype=torch.complex64, device=P.device)
    _check(lib().chain_txrx_ex(_ptr(P), _ptr(s_tilde), _ptr(coef), _ptr(y), _ptr(XPA), _ints(orders), len(orders),
                               L, M, n_sym, B, U, N_d, N_ifft, C.byref(imp), _stream(P)))
    return y, XPA


def ue_combine_ser_ex(XPA, h_fd, alpha, tx_idx, M_qam, imp, yhat=None, counts=None, dec=None, boundary_eps=1e-4):
    """ue_combine_ser with AWGN at the UEs (imp.awgn_n0)."""
    _dev(XPA, torch.complex64, "XPA")
    _dev(h_fd, torch.complex64, "h_fd")
    _dev(tx_idx, torch.uint16, "tx_idx")
    n_sym, B, N_d = XPA.shape
    U = h_fd.shape[0]
    if yhat is None:
        yhat = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=XPA.device)
    if counts is None:
        counts = torch.zeros(3, dtype=torch.int64, device=XPA.device)
    _check(lib().ue_combine_ser_ex(_ptr(XPA), _ptr(h_fd), _ptr(yhat), float(alpha), _ptr(tx_idx), M_qam, _ptr(dec),
                                   _ptr(counts), n_sym, B, U, N_d, float(boundary_eps), C.byref(imp), _stream(XPA)))
    return yhat, counts, dec


def chain_txrx(P, s_tilde, coef, orders, L, M, N_ifft, y=None, XPA=None):
    """Fused precode -> IDFT -> GMP -> receive DFT.  Returns (y [n_sym][B_loc][N_ifft], XPA [n_sym][B_loc][N_d])."""
    _dev(P, torch.complex64, "P")
    _dev(s_tilde, torch.complex64, "s_tilde")
    _dev(coef, torch.complex64, "coef")
    B, U, N_d = P.shape
    n_sym = s_tilde.shape[0]
    if y is None:
        y = torch.empty((n_sym, B, N_ifft), dtype=torch.complex64, device=P.device)
    if XPA is None:
        XPA = torch.empty((n_sym, B, N_d), dtype=torch.complex64, device=P.device)
    _check(lib().chain_txrx(_ptr(P), _ptr(s_tilde), _ptr(coef), _ptr(y), _ptr(XPA),
                            _ints(orders), len(orders), L, M, n_sym, B, U, N_d, N_ifft, _stream(P)))
    return y, XPA


# ----------------------------------------------------------------------------- a6
def ue_combine(XPA, h_fd, out=None, accumulate=False):
    _dev(XPA, torch.complex64, "XPA")
    _dev(h_fd, torch.complex64, "h_fd")
    n_sym, B, N_d = XPA.shape
    U = h_fd.shape[0]
    if out is None:
        out = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=XPA.device)
    _check(lib().ue_combine(_ptr(XPA), _ptr(h_fd), _ptr(out), n_sym, B, U, N_d, int(bool(accumulate)),
                            _stream(XPA)))
    return out


def ue_combine_peer(XPA, h_fd, peer_recv, rank):
    """Mode A: the channel sum over this rank's antennas with every partial y_hat stored straight
    into slot `rank` of its owner's receive buffer (include/fdpd.h ue_combine_peer).  XPA
    [world * nm][B_loc][N_d]; peer_recv: list of `world` tensors [world][nm][U][N_d] complex64,
    entry r the (peer-mapped) receive buffer of rank r."""
    _dev(XPA, torch.complex64, "XPA")
    _dev(h_fd, torch.complex64, "h_fd")
    n_sym, B, N_d = XPA.shape
    U = h_fd.shape[0]
    ws = len(peer_recv)
    if n_sym % ws:
        raise ValueError(f"ue_combine_peer: {n_sym} symbols do not split over {ws} ranks")
    for t in peer_recv:
        _dev(t, torch.complex64, "peer_recv")
        if tuple(t.shape) != (ws, n_sym // ws, U, N_d):
            raise ValueError(f"ue_combine_peer: receive buffer {tuple(t.shape)} != {(ws, n_sym // ws, U, N_d)}")
    ptrs = (C.c_void_p * ws)(*[t.data_ptr() for t in peer_recv])
    _check(lib().ue_combine_peer(_ptr(XPA), _ptr(h_fd), ptrs, ws, int(rank), n_sym, B, U, N_d, _stream(XPA)))


def ue_reduce_ser(recv, alpha=1.0, tx_idx=None, M_qam=4, yhat=None, counts=None, dec=None, boundary_eps=1e-4):
    """Mode A, owner side: y_hat = sum of the `world` slots of recv [world][n][U][N_d] in rank order,
    then slicing + SER when tx_idx is given (include/fdpd.h ue_reduce_ser).  Returns (yhat, counts, dec)."""
    _dev(recv, torch.complex64, "recv")
    ws, n_sym, U, N_d = recv.shape
    if yhat is None:
        yhat = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=recv.device)
    if tx_idx is not None:
        _dev(tx_idx, torch.uint16, "tx_idx")
        if counts is None:
            counts = torch.zeros(3, dtype=torch.int64, device=recv.device)
    _check(lib().ue_reduce_ser(_ptr(recv), ws, _ptr(yhat), float(alpha), _ptr(tx_idx), int(M_qam), _ptr(dec),
                               _ptr(counts), n_sym, U, N_d, float(boundary_eps), _stream(recv)))
    return yhat, counts, dec


def ue_combine_ser(XPA, h_fd, alpha, tx_idx, M_qam, yhat=None, counts=None, dec=None, boundary_eps=1e-4):
    _dev(XPA, torch.complex64, "XPA")
    _dev(h_fd, torch.complex64, "h_fd")
    _dev(tx_idx, torch.uint16, "tx_idx")
    n_sym, B, N_d = XPA.shape
    U = h_fd.shape[0]
    if yhat is None:
        yhat = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=XPA.device)
    if counts is None:
        counts = torch.zeros(3, dtype=torch.int64, device=XPA.device)
    _check(lib().ue_combine_ser(_ptr(XPA), _ptr(h_fd), _ptr(yhat), float(alpha), _ptr(tx_idx), M_qam, _ptr(dec),
                                _ptr(counts), n_sym, B, U, N_d, float(boundary_eps), _stream(XPA)))
    return yhat, counts, dec

def ue_receive(y, h_fd, out=None, accumulate=False, workspace=None):
    _dev(y, torch.complex64, "y")
    _dev(h_fd, torch.complex64, "h_fd")
    n_sym, B, N = y.shape
    U, _, N_d = h_fd.shape
    if out is None:
        out = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=y.device)
    need = lib().ue_receive_workspace_bytes(n_sym, B, N_d)
    if workspace is None or workspace.numel() < need:
        workspace = _ws(need, y)
    _check(lib().ue_receive(_ptr(y), _ptr(h_fd), _ptr(out), _ptr(workspace), workspace.numel(), n_sym, B, U, N_d, N,
                            int(bool(accumulate)), _stream(y)))
    return out


def ue_slice_ser(yhat, alpha, tx_idx, M_qam, counts=None, dec=None, boundary_eps=1e-4):
    """Returns counts (device int64[3]: errors, total, near) and dec (uint16 or None)."""
    _dev(yhat, torch.complex64, "yhat")
    _dev(tx_idx, torch.uint16, "tx_idx")
    n_sym, U, N_d = yhat.shape
    if counts is None:
        counts = torch.zeros(3, dtype=torch.int64, device=yhat.device)
    _check(lib().ue_slice_ser(_ptr(yhat), float(alpha), _ptr(tx_idx), M_qam, _ptr(dec), _ptr(counts), n_sym, U, N_d,
                              float(boundary_eps), _stream(yhat)))
    return counts, dec


def ue_receive_ser(y, h_fd, alpha, tx_idx, M_qam, yhat=None, counts=None, dec=None, workspace=None,
                   boundary_eps=1e-4):
    _dev(y, torch.complex64, "y")
    _dev(h_fd, torch.complex64, "h_fd")
    _dev(tx_idx, torch.uint16, "tx_idx")
    n_sym, B, N = y.shape
    U, _, N_d = h_fd.shape
    if yhat is None:
        yhat = torch.empty((n_sym, U, N_d), dtype=torch.complex64, device=y.device)
    if counts is None:
        counts = torch.zeros(3, dtype=torch.int64, device=y.device)
    need = lib().ue_receive_workspace_bytes(n_sym, B, N_d)
    if workspace is None or workspace.numel() < need:
        workspace = _ws(need, y)
    _check(lib().ue_receive_ser(_ptr(y), _ptr(h_fd), _ptr(yhat), _ptr(workspace), workspace.numel(), float(alpha),
                                _ptr(tx_idx), M_qam, _ptr(dec), _ptr(counts), n_sym, B, U, N_d, N,
                                float(boundary_eps), _stream(y)))
    return yhat, counts, dec


# ----------------------------------------------------------------------------- native runtime
class NativeChain:
    """The C runtime plan (fd_chain_*): device-resident state of one channel realisation;
    run_host() is the end-to-end entry point (host inputs in, SER counters out)."""

    def __init__(self, cfg_shapes, h_taps, coef, params, max_batch, device=None):
        import numpy as np
        sh = cfg_shapes
        d = ChainDesc()
        d.U, d.B, d.T = sh.U, sh.B, int(np.asarray(h_taps).shape[0])
        d.N_d, d.N_ifft, d.M_qam = sh.N_d, sh.N_ifft, sh.M_qam
        d.n_layers = len(sh.chans) - 1
        for i, c in enumerate(sh.chans):
            d.chans[i] = c
        d.n_orders = len(sh.orders)
        for i, o in enumerate(sh.orders):
            d.orders[i] = o
        d.L, d.M, d.rho, d.boundary_eps = sh.L, sh.M, sh.rho, sh.eps
        d.head, d.n_conv = (1 if getattr(sh, "head", "residual") == "paper" else 0), getattr(sh, "n_conv", 2)
        self.desc = d
        self.device = torch.device("cuda") if device is None else torch.device(device)
        self._keep = [np.ascontiguousarray(h_taps, dtype=np.complex64), np.ascontiguousarray(coef, dtype=np.complex64),
                      np.ascontiguousarray(params, dtype=np.float32)]
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
            _check(lib().fd_chain_create(C.byref(h), C.byref(d), self._keep[0].ctypes.data, self._keep[1].ctypes.data,
                                         self._keep[2].ctypes.data, int(max_batch), st))
        self.h = h
        self.alpha = float(lib().fd_chain_alpha(h))

    def run_device(self, s, tx_idx, counts, yhat=None):
        _dev(s, torch.complex64, "s")
        _dev(tx_idx, torch.uint16, "tx_idx")
        _check(lib().fd_chain_run_device(self.h, _ptr(s), _ptr(tx_idx), s.shape[0], _ptr(counts), _ptr(yhat),
                                         _stream(s)))
        return counts

    def run_host(self, s_host, idx_host, counts_host):
        """s_host, idx_host, counts_host: (pinned) CPU tensors; returns counts_host."""
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().fd_chain_run_host(self.h, C.c_void_p(s_host.data_ptr()), C.c_void_p(idx_host.data_ptr()),
                                       s_host.shape[0], C.c_void_p(counts_host.data_ptr()), st))
        return counts_host

    def run_host_qam(self, idx_host, counts_host):
        """idx_host, counts_host: (pinned) CPU tensors; the QAM mapping runs on the device."""
        st = C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)
        _check(lib().fd_chain_run_host_qam(self.h, C.c_void_p(idx_host.data_ptr()), idx_host.shape[0],
                                           C.c_void_p(counts_host.data_ptr()), st))
        return counts_host

    def close(self):
        if getattr(self, "h", None) is not None and self.h.value:
            lib().fd_chain_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

"""C-ABI checks that need no GPU: libfdpd.so loads, exports every entry point that
include/fdpd.h declares, the Python binding mirrors them, and argument validation
fails with FD_ERR_ARG before any CUDA call."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "fdpd.h")
LIB = os.path.join(ROOT, "paper_2205_05158_b200", "libfdpd.so")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:const\s+)?[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n not in ("if", "while")))


@pytest.fixture(scope="module")
def lib():
    if not os.path.exists(LIB):
        from paper_2205_05158_b200 import build
        build.build()
    return ctypes.CDLL(LIB)


def test_header_declares_the_section8_boundary():
    names = declared_functions()
    for fn in ["fdcnn_forward", "zf_precoder_build", "precode", "ofdm_modulate", "gmp_pa", "chain_tx",
               "ue_receive", "ue_slice_ser", "ue_receive_ser", "fd_last_error"]:
        assert fn in names


def test_every_declared_symbol_is_exported(lib):
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_mirrors_header():
    from paper_2205_05158_b200 import fdpd
    assert set(fdpd.SIGNATURES) == set(declared_functions())


def test_argument_errors_without_gpu(lib):
    lib.fd_last_error.restype = ctypes.c_char_p
    f = lib.ofdm_modulate
    f.restype = ctypes.c_int
    f.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                  ctypes.c_void_p]
    assert f(None, None, 1, 1, 36, 128, None) == 2
    assert b"NULL" in lib.fd_last_error()
    buf = (ctypes.c_byte * 64)()
    p = ctypes.cast(buf, ctypes.c_void_p).value
    p16 = (p + 15) // 16 * 16
    assert f(p16, p16, 1, 1, 36, 100, None) == 2          # not a power of two
    assert b"power of two" in lib.fd_last_error()
    assert f(p16, p16, 1, 1, 37, 128, None) == 2          # odd N_d
    g = lib.gmp_pa
    g.restype = ctypes.c_int
    orders = (ctypes.c_int * 2)(1, 4)
    g.argtypes = [ctypes.c_void_p] * 3 + [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                          ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_void_p]
    assert g(p16, p16, p16 + 16, orders, 2, 1, 1, 1, 1, 64, None) == 2   # even order
    assert b"odd" in lib.fd_last_error()
    assert g(p16, p16, p16, orders, 2, 1, 1, 1, 1, 64, None) == 2        # aliasing
    z = lib.zf_precoder_build
    z.restype = ctypes.c_int
    assert lib.fd_version() == 100


def test_workspace_queries(lib):
    lib.ue_receive_workspace_bytes.restype = ctypes.c_size_t
    lib.ue_receive_workspace_bytes.argtypes = [ctypes.c_longlong, ctypes.c_int, ctypes.c_int]
    assert lib.ue_receive_workspace_bytes(1024, 64, 600) == 8 * 1024 * 64 * 600
    lib.fdcnn_workspace_bytes.restype = ctypes.c_size_t
    lib.fdcnn_workspace_bytes.argtypes = [ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.c_longlong,
                                          ctypes.c_int, ctypes.c_int]
    lib.fd_set_cnn_path.restype = ctypes.c_int
    lib.fd_set_cnn_path.argtypes = [ctypes.c_int]
    assert lib.fd_set_cnn_path(7) == 2                                   # unknown path: FD_ERR_ARG
    try:
        assert lib.fd_set_cnn_path(1) == 0                               # SIMT kernels
        ch = (ctypes.c_int * 4)(2, 16, 16, 2)
        assert lib.fdcnn_workspace_bytes(ch, 3, 1024, 4, 600) == 0      # C2: whole network in shared memory
        ch = (ctypes.c_int * 5)(2, 32, 32, 32, 2)
        act = 2 * 4 * 16 * 8 * 32 * 35 * 35                  # C3: per-layer, two activation buffers
        assert act < lib.fdcnn_workspace_bytes(ch, 4, 16, 8, 1200) < act + (1 << 20)   # + transposed weights
        assert lib.fd_set_cnn_path(2) == 0                               # tensor cores
        # two activation buffers of PP pixels x 32 channels x 4 B per image: PP = the split-fp16
        # plane length (conv_tc.cu tc_geom: 8 guard pixels + (n_tiles - 1) * 128 + A_px + 8, rounded
        # to 8) >= the (S + 2)^2 haloed pixels of the TF32 mode's channels-last layout
        S, Wp = 35, 37
        n_tiles, A_px = (S * Wp + 127) // 128, (128 + 2 * Wp + 2 + 7) & ~7
        PP = (8 + max(Wp * Wp, (n_tiles - 1) * 128 + A_px) + 8 + 7) & ~7
        act = 2 * 4 * 16 * 8 * 32 * PP
        wsplit = 4 * 9 * 2 * (8 * 32 + 32 * 32 * 2 + 32 * 16)   # hi/lo weight images, padded
        tc_bytes = lib.fdcnn_workspace_bytes(ch, 4, 16, 8, 1200)
        assert act + wsplit <= tc_bytes < act + wsplit + 4096
        assert lib.fd_set_cnn_path(0) == 0                               # auto: tensor cores from width 32
        assert lib.fdcnn_workspace_bytes(ch, 4, 16, 8, 1200) == tc_bytes
        assert lib.fdcnn_workspace_bytes((ctypes.c_int * 4)(2, 16, 16, 2), 3, 1024, 4, 600) == 0
    finally:
        lib.fd_set_cnn_path(0)

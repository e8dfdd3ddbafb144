"""B200-native hot path of the FD-CNN DPD massive MU-MIMO-OFDM downlink (arXiv 2205.05158).

The compute lives in ``libfdpd.so`` (hand-written sm_100a CUDA behind a C ABI,
``include/fdpd.h``); ``paper_2205_05158_b200.fdpd`` is a thin ctypes binding with
the same entry-point names.  There is no CPU fallback: every call fails loudly if
the library is missing or the device is not CUDA.
"""
__all__ = ["fdpd"]

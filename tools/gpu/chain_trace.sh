#!/bin/bash
# Per-CTA phase timeline of the C5 chain kernel (build first: tools/build_variant.sh
# variants/libfdpd_trace.so "-DFD_TRACE=1" chain_cl.cu).  FD_OCC1=1: one CTA per SM.
FDPD_LIB=$PWD/variants/libfdpd_trace.so timeout 300 python tools/chain_trace.py > gpurun_out/chain_trace.txt 2>&1

#!/bin/bash
FD_OCC1=1 FDPD_LIB=$PWD/variants/libfdpd_trace.so timeout 300 python tools/chain_trace.py > gpurun_out/s4_trace_occ1.txt 2>&1

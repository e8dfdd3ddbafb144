#!/bin/bash
# quick chain timing + phase trace (variants/libfdpd_trace.so built with -DFD_TRACE=1)
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/chain_quick_c5.json 2> gpurun_out/chain_quick_c5.err
[ -f variants/libfdpd_trace.so ] && FDPD_LIB=$PWD/variants/libfdpd_trace.so timeout 300 python tools/chain_trace.py > gpurun_out/chain_trace.txt 2>&1
timeout 600 python -m pytest tests -m gpu -q -x -k "cluster or gmp_tc or guard_chain" 2>&1 | tail -3 > gpurun_out/chain_quick_tests.log

#!/bin/bash
B="python bench.py --no-cpu-baseline --steps 1 --warmup 3"
timeout 300 $B > gpurun_out/combine_prof_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_rx_combine_tile -s 3 -c 1 \
  -o gpurun_out/combine_prof -f $B > gpurun_out/combine_prof_ncu.log 2>&1
timeout 600 python -m pytest tests/test_gpu_combine_tc.py -q -x 2>&1 | tail -3 > gpurun_out/s4_comb_tests2.log

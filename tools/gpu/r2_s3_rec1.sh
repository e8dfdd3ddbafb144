#!/bin/bash
# record: full GPU suite, C5 default + fp32tc + combine simt, C2/C3/C4 lines
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/rec1_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/rec1_c5.json 2>&1
$B --precode-math fp32tc > gpurun_out/rec1_c5_fp32tc.json 2>&1
$B --precode-math fp32tc --combine simt > gpurun_out/rec1_c5_fp32tc_csimt.json 2>&1
for c in C2 C3 C4; do $B --config $c > gpurun_out/rec1_$c.json 2>&1; done
$B --config C3 --split-precode --precode-math tf32 > gpurun_out/rec1_C3_tf32.json 2>&1

#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_guard.py tests/test_gpu_parity.py tests/test_gpu_precode_tc.py tests/test_gpu_combine_tc.py -q -x -k "guard or fdcnn or end_to_end_large or native or precode or combine" 2>&1 | tail -15 > gpurun_out/e4_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B --precode-math fp32tc > gpurun_out/e4_fp32tc.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_conv|k_combine_tc|k_precode_tc" -s 7 -c 6 -o gpurun_out/e4_prof -f python bench.py --no-cpu-baseline --steps 1 --warmup 1 --precode-math fp32tc > gpurun_out/e4_ncu.log 2>&1

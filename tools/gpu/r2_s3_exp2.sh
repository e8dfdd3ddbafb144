#!/bin/bash
# combine (strided quads) + tap7: tests, C5 bench, CNN / combine ncu, memcheck of the sanitizer cases
timeout 900 python -m pytest tests/test_gpu_combine_tc.py tests/test_gpu_parity.py -q -x -k "combine or end_to_end or random or chain" 2>&1 | tail -3 > gpurun_out/e2_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/e2_base.json 2>&1
$B --precode-math fp32tc > gpurun_out/e2_fp32tc.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_conv|k_combine_tc" -s 12 -c 6 -o gpurun_out/e2_cnn -f python bench.py --no-cpu-baseline --steps 1 --warmup 2 --precode-math fp32tc > gpurun_out/e2_ncu.log 2>&1
timeout 900 compute-sanitizer --tool memcheck --leak-check no python tools/sanitize_cases.py > gpurun_out/e2_memcheck.log 2>&1; echo "rc=$?" >> gpurun_out/e2_memcheck.log

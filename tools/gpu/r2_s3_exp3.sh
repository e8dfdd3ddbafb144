#!/bin/bash
# ACT16 CNN: guard + CNN parity tests, C5 bench, CNN ncu
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_parity.py -q -x -k "guard or fdcnn or end_to_end_large or native" 2>&1 | tail -15 > gpurun_out/e3_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B --precode-math fp32tc > gpurun_out/e3_fp32tc.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_conv" -s 5 -c 3 -o gpurun_out/e3_cnn -f python bench.py --no-cpu-baseline --steps 1 --warmup 1 --precode-math fp32tc > gpurun_out/e3_ncu.log 2>&1

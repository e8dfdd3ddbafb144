#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_gmp_tc.py tests/test_gpu_guard.py -q -x -k "gmp or chain" 2>&1 | tail -4 > gpurun_out/e11_tests.log
timeout 300 python tools/tcg_check3.py C5 > gpurun_out/e11_det.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --gmp tc > gpurun_out/e11_c5_tc.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_chain_cl" -c 1 -o gpurun_out/e11_chain_tc -f python bench.py --no-cpu-baseline --steps 1 --warmup 1 --gmp tc > /dev/null 2>&1

#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_gmp_tc.py tests/test_gpu_guard.py -q -x 2>&1 | tail -4 > gpurun_out/e10_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 --gmp tc > gpurun_out/e10_c5_tc.json 2>&1
timeout 300 python bench.py --config C4 --no-cpu-baseline --steps 10 --warmup 3 --gmp tc > gpurun_out/e10_c4_tc.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_chain_cl" -c 1 -o gpurun_out/e10_chain_tc -f python bench.py --no-cpu-baseline --steps 1 --warmup 1 --gmp tc > /dev/null 2>&1

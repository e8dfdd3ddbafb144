#!/bin/bash
# tensor-core GMP v4: parity tests, guard/poison checks, bench lines (tc vs simt)
timeout 900 python -m pytest tests/test_gpu_gmp_tc.py -q -x -s 2>&1 | tail -25 > gpurun_out/s4_tc_tests.log
timeout 600 python -m pytest tests/test_gpu_guard.py -q -x -k chain 2>&1 | tail -5 >> gpurun_out/s4_tc_tests.log
timeout 300 python tools/tcg_check3.py C5 > gpurun_out/s4_tc_poison.log 2>&1
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B --gmp tc > gpurun_out/s4_tc_bench.json 2> gpurun_out/s4_tc_bench.err
$B --gmp simt > gpurun_out/s4_simt_bench.json 2> gpurun_out/s4_simt_bench.err

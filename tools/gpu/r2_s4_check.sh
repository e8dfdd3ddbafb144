#!/bin/bash
# Session 4 first check after container re-creation: full GPU suite, default C5 line, C2 line.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s4_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s4_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s4_bench_c5.json 2> gpurun_out/s4_bench_c5.err
timeout 600 python bench.py --no-cpu-baseline --config C2 > gpurun_out/s4_bench_c2.json 2> gpurun_out/s4_bench_c2.err

#!/bin/bash
# Session 3 first check: full GPU suite, default C5 line, fp32tc precode line, stage timings.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/s3_smi.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/s3_gpu_tests.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/s3_bench_c5.json 2> gpurun_out/s3_bench_c5.err
timeout 600 python bench.py --no-cpu-baseline --precode-math fp32tc > gpurun_out/s3_bench_c5_fp32tc.json 2> gpurun_out/s3_bench_c5_fp32tc.err
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C5 32 10 > gpurun_out/s3_stage_c5.json 2>&1

set -x
timeout 600 python -m pytest tests/test_gpu_precode_tc.py -x -q 2>&1 | tail -15 > gpurun_out/r2_precode_tests.log
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C5 32 10 > gpurun_out/r2_stage_precode_c5.json 2>&1
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C3 512 10 > gpurun_out/r2_stage_precode_c3.json 2>&1
timeout 900 python -m pytest tests/test_gpu_modeA.py -x -q 2>&1 | tail -30 > gpurun_out/r2_modeA_tests.log
timeout 300 python bench.py --no-cpu-baseline --precode-math fp32tc > gpurun_out/r2_bench_c5_fp32tc.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --mode antenna --precode-math fp32tc > gpurun_out/r2_bench_c5_modeA1.json 2>&1

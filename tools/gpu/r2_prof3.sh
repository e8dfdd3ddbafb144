set -x
timeout 900 python -m pytest tests/test_gpu_precode_tc.py tests/test_gpu_parity.py -x -q -k "precode or chain or end_to_end_large or random" 2>&1 | tail -5 > gpurun_out/r2_tests_p3.log
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C5 32 10 > gpurun_out/r2_stage_precode_c5.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --precode-math fp32tc > gpurun_out/r2_bench_c5_v3.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --precode-math fp32tc --steps 1 --warmup 1 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv_tc<64|k_combine_tc|k_chain_cl|k_precode_tc" -c 6 -o gpurun_out/r2_c5_all -f python bench.py --no-cpu-baseline --precode-math fp32tc --steps 1 --warmup 1 > gpurun_out/ncu3.log 2>&1

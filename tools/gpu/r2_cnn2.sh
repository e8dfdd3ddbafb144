set -x
timeout 900 python -m pytest tests/test_gpu_combine_tc.py tests/test_gpu_parity.py -x -q -k "combine or fdcnn or end_to_end_large" 2>&1 | tail -15 > gpurun_out/r2_tests_cnn2.log
STAGES=fdcnn_forward timeout 300 python tools/stage_bench.py C5 32 10 > gpurun_out/r2_stage_cnn_c5.json 2>&1
STAGES=fdcnn_forward timeout 300 python tools/stage_bench.py C4 128 10 > gpurun_out/r2_stage_cnn_c4.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --precode-math fp32tc > gpurun_out/r2_bench_c5_v2.json 2>&1
timeout 300 python tools/cnn_one.py C5 32 > gpurun_out/plain_cnn.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cnn_launches_c5.csv python tools/cnn_one.py C5 32 > /dev/null 2>&1
STAGES=precode_fp32tc timeout 300 python tools/stage_bench.py C5 32 3 > gpurun_out/plain_pc.log 2>&1 && \
STAGES=precode_fp32tc timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_precode_tc -s 2 -c 1 -o gpurun_out/r2_precode_c5c -f python tools/stage_bench.py C5 32 3 > gpurun_out/ncu_pc.log 2>&1

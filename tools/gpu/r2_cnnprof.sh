set -x
timeout 600 python -m pytest tests/test_gpu_precode_tc.py -x -q 2>&1 | tail -5 > gpurun_out/r2_precode_tests.log
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C5 32 10 > gpurun_out/r2_stage_precode_c5.json 2>&1
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C3 512 10 > gpurun_out/r2_stage_precode_c3.json 2>&1
timeout 300 python tools/cnn_one.py C5 32 > gpurun_out/plain_cnn.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_cnn_launches_c5.csv python tools/cnn_one.py C5 32 > /dev/null 2>&1 ; \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_conv -s 0 -c 6 -o gpurun_out/r2_cnn_c5 -f python tools/cnn_one.py C5 32 > gpurun_out/ncu_cnn.log 2>&1

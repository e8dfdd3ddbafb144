set -x
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/r2_gpu_tests.log
STAGES=fdcnn_forward timeout 300 python tools/stage_bench.py C5 32 10 > gpurun_out/r2_stage_cnn_c5.json 2>&1
STAGES=fdcnn_forward timeout 300 python tools/stage_bench.py C4 128 10 > gpurun_out/r2_stage_cnn_c4.json 2>&1
STAGES=fdcnn_forward timeout 300 python tools/stage_bench.py C3 512 10 > gpurun_out/r2_stage_cnn_c3.json 2>&1
timeout 300 python bench.py --no-cpu-baseline --precode-math fp32tc > gpurun_out/r2_bench_c5_f16.json 2>&1
STAGES=precode_fp32tc timeout 300 python tools/stage_bench.py C5 32 3 > gpurun_out/plain_pc.log 2>&1 && \
STAGES=precode_fp32tc timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_precode_tc -s 2 -c 1 -o gpurun_out/r2_precode_c5b -f python tools/stage_bench.py C5 32 3 > gpurun_out/ncu_pc.log 2>&1

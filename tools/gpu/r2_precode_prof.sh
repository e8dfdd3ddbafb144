set -x
STAGES=precode_fp32tc timeout 300 python tools/stage_bench.py C5 32 3 > gpurun_out/plain_pc.log 2>&1 && \
STAGES=precode_fp32tc timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_precode_tc -s 2 -c 1 -o gpurun_out/r2_precode_c5 -f python tools/stage_bench.py C5 32 3 > gpurun_out/ncu_pc.log 2>&1

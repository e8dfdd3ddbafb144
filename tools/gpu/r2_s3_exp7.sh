#!/bin/bash
CNN_TIME_TENSOR_ONLY=1 timeout 300 python tools/cnn_time.py C5:32 C4:128 C3:512 > gpurun_out/e7_cnn.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_guard.py tests/test_gpu_parity.py -q -x -k "guard or fdcnn or end_to_end" 2>&1 | tail -4 > gpurun_out/e7_tests.log
timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/e7_c5.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:k_conv_tc" -s 4 -c 2 -o gpurun_out/e7_cnn -f python bench.py --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1

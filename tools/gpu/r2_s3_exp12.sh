#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_guard.py -q -x -k "fdcnn" 2>&1 | tail -3 > gpurun_out/e12_tests.log
CNN_TIME_TENSOR_ONLY=1 timeout 300 python tools/cnn_time.py C5:32 C4:128 C3:512 > gpurun_out/e12_cnn.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3 > gpurun_out/e12_c5.json 2>&1

#!/bin/bash
# CNN weight ring vs resident
for w in 0 4 6 9; do echo "wring=$w"; CNN_TIME_TENSOR_ONLY=1 FDPD_TC_WRING=$w timeout 300 python tools/cnn_time.py C5:32 C4:128 C3:512; done > gpurun_out/e5_cnn.log 2>&1

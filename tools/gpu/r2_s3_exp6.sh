#!/bin/bash
for d in 0 1; do echo "dbg=$d"; CNN_TIME_TENSOR_ONLY=1 FDPD_TC_DBG=$d timeout 300 python tools/cnn_time.py C5:32 C4:128; done > gpurun_out/e6_cnn.log 2>&1
timeout 600 ncu --set full --clock-control none -k "regex:k_conv_tc<64, 64, 0, 2" -c 1 -o gpurun_out/e6_cnn_dbg1 -f env FDPD_TC_DBG=1 CNN_TIME_TENSOR_ONLY=1 python tools/cnn_time.py C5:32 > /dev/null 2>&1

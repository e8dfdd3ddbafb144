#!/bin/bash
# ncu --set full + source of the FD-CNN kernels of one C5 forward (tools/cnn_one.py)
timeout 300 python tools/cnn_one.py C5 32 > gpurun_out/cnn_prof_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_conv" -s 0 -c 5 -o gpurun_out/cnn_prof -f python tools/cnn_one.py C5 32 > gpurun_out/cnn_prof_ncu.log 2>&1

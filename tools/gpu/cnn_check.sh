#!/bin/bash
# CNN change check: FD-CNN parity / guard tests, C5 / C4 / C3 bench lines
timeout 1200 python -m pytest tests -m gpu -q -x -k "cnn or guard or end_to_end or native" 2>&1 | tail -5 > gpurun_out/cnn_check_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/cnn_check_c5.json 2>&1
$B --config C4 > gpurun_out/cnn_check_c4.json 2>&1
$B --config C3 > gpurun_out/cnn_check_c3.json 2>&1

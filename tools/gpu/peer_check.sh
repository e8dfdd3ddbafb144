#!/bin/bash
# fused Mode A exchange: single-GPU parity, 2-rank IPC validation, Mode A bench path at 1 rank
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "combine" 2>&1 | tail -5 > gpurun_out/peer_check_tests.log
timeout 1500 python -m pytest tests/test_gpu_modeA.py -q -x 2>&1 | tail -8 >> gpurun_out/peer_check_tests.log
timeout 300 python bench.py --no-cpu-baseline --mode antenna --steps 5 --warmup 3 > gpurun_out/peer_check_modeA.json 2> gpurun_out/peer_check_modeA.err
timeout 300 python bench.py --no-cpu-baseline --steps 5 --warmup 3 > gpurun_out/peer_check_c5.json 2> gpurun_out/peer_check_c5.err

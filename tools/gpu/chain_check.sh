#!/bin/bash
# chain kernel change check: chain / GMP / guard / end-to-end parity tests, C5 and C4 bench lines
timeout 1500 python -m pytest tests -m gpu -q -x -k "chain or gmp or guard or end_to_end or e2e or random" 2>&1 | tail -6 > gpurun_out/chain_check_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/chain_check_c5.json 2> gpurun_out/chain_check_c5.err
$B --config C4 > gpurun_out/chain_check_c4.json 2> gpurun_out/chain_check_c4.err

#!/bin/bash
# chain kernel change check: chain parity/guard/gmp_tc tests, C5 + C4 bench lines (simt and tc)
timeout 1200 python -m pytest tests -m gpu -q -x -k "chain or gmp or guard or end_to_end or e2e" 2>&1 | tail -6 > gpurun_out/s4_chain_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/s4_chain_c5.json 2> gpurun_out/s4_chain_c5.err
$B --gmp tc > gpurun_out/s4_chain_c5_tc.json 2> gpurun_out/s4_chain_c5_tc.err
$B --config C4 > gpurun_out/s4_chain_c4.json 2> gpurun_out/s4_chain_c4.err

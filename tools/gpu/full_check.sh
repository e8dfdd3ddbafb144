#!/bin/bash
# full GPU suite + the bench lines of C2..C5
timeout 2400 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/full_check_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
for c in C5 C4 C3 C2; do $B --config $c > gpurun_out/full_check_$c.json 2>&1; done

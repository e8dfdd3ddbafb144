#!/bin/bash
timeout 1200 python -m pytest tests -m gpu -q -x -k "combine or guard or end_to_end or ser or impair or redraw or modeA or native" 2>&1 | tail -6 > gpurun_out/combine_check_tests.log
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/combine_check_c5.json 2> gpurun_out/combine_check_c5.err
$B --config C4 > gpurun_out/combine_check_c4.json 2> gpurun_out/combine_check_c4.err
$B --config C3 > gpurun_out/combine_check_c3.json 2> gpurun_out/combine_check_c3.err

#!/bin/bash
# Session-4 record: full GPU suite, bench lines of every config and variant, reference arm,
# C5 launch list, ncu --set full of the C5 step's kernels, stage timings.
O=gpurun_out/r2s4
mkdir -p $O /tmp/reps
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > $O/smi.txt
timeout 2400 python -m pytest tests -m gpu -q 2>&1 | tail -6 > $O/gpu_tests.txt
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/reference_c5.json 2> $O/reference_c5.err
B="timeout 400 python bench.py --no-cpu-baseline"
for c in C1 C2 C3 C4 P; do $B --config $c > $O/bench_$c.json 2> $O/bench_$c.err; done
$B --config C3 --split-precode --precode-math tf32 > $O/bench_C3_tf32.json 2>&1
$B --config C2 --impair > $O/bench_C2_impair.json 2>&1
$B --config C2 --redraw --steps 10 > $O/bench_C2_redraw.json 2>&1
$B --config C2 --unfused > $O/bench_C2_unfused.json 2>&1
$B --gmp tc > $O/bench_c5_gmp_tc.json 2>&1
$B --combine tc > $O/bench_c5_combine_tc.json 2>&1
$B --precode-math simt > $O/bench_c5_precode_simt.json 2>&1
$B --mode antenna > $O/bench_c5_modeA_1rank.json 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_chain_cl|k_precode_tc|k_rx_combine|k_conv_tc|k_conv_out" -s 12 -c 7 -o /tmp/reps/c5 -f \
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline > $O/ncu_c5.log 2>&1
python tools/ncu_summary.py /tmp/reps/c5.ncu-rep > $O/ncu_c5_summary.txt 2>&1
ncu -i /tmp/reps/c5.ncu-rep --page raw --csv > $O/ncu_c5_raw.csv 2>/dev/null
timeout 600 python tools/stage_bench.py C5 32 10 > $O/stage_c5.json 2>&1
echo done > $O/DONE

#!/bin/bash
# C5 / C4 default lines, the C5 launch list and ncu --set full of the C5 step's kernels.
T=${1:-r2}
O=gpurun_out/$T
mkdir -p $O /tmp/reps
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 400 python bench.py --no-cpu-baseline --config C4 > $O/bench_C4.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --gmp tc > $O/bench_c5_gmp_tc.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --combine tc > $O/bench_c5_combine_tc.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --precode-math simt > $O/bench_c5_precode_simt.json 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_chain_cl|k_precode_tc|k_rx_combine|k_conv_tc|k_conv_out" -s 12 -c 7 -o /tmp/reps/c5 -f \
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline > $O/ncu_c5.log 2>&1
python tools/ncu_summary.py /tmp/reps/c5.ncu-rep > $O/ncu_c5_summary.txt 2>&1
ncu -i /tmp/reps/c5.ncu-rep --page raw --csv > $O/ncu_c5_raw.csv 2>/dev/null
echo done > $O/DONE

#!/bin/bash
# Round-2 record run: GPU tests, bench lines (C5 default with the all-core oracle baseline, the
# reference arm, C1-C4, P, the C3 TF32 variant, impairments, per-symbol redraw, unfused, the
# tensor-core GMP opt-in), stage timings, the C5 launch list and ncu --set full captures of the
# C5 step's kernels (summaries + raw CSV; the .ncu-rep files stay on the box).
# usage: bash tools/gpu/r2_record.sh TAG
T=${1:-r2}
O=gpurun_out/$T
mkdir -p $O /tmp/reps
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1800 python -m pytest tests -m gpu -q 2>&1 | tail -5 > $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_c5.json 2> $O/bench_c5.err
timeout 1200 python bench.py --impl reference > $O/reference_c5.json 2> $O/reference_c5.err
for c in C1 C2 C3 C4 P; do timeout 400 python bench.py --no-cpu-baseline --config $c > $O/bench_$c.json 2>&1; done
timeout 400 python bench.py --no-cpu-baseline --config C3 --split-precode --precode-math tf32 > $O/bench_C3_tf32.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --config C2 --impair > $O/bench_C2_impair.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --config C2 --redraw --steps 10 > $O/bench_C2_redraw.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --config C2 --unfused > $O/bench_C2_unfused.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --gmp tc > $O/bench_c5_gmp_tc.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --combine tc > $O/bench_c5_combine_tc.json 2>&1
timeout 400 python bench.py --no-cpu-baseline --precode-math simt > $O/bench_c5_precode_simt.json 2>&1
STAGES=precode,precode_fp32tc,precode_tf32 timeout 300 python tools/stage_bench.py C5 32 10 > $O/stage_c5.json 2>&1
timeout 300 python tools/stage_bench.py C2 1024 10 > $O/stage_c2.json 2>&1
CNN_TIME_TENSOR_ONLY=1 timeout 300 python tools/cnn_time.py C5:32 C4:128 C3:512 > $O/cnn_time.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/plain.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file $O/launches_c5.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline > $O/ncu_launch.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on \
  -k regex:"k_chain_cl|k_precode_tc|k_rx_combine|k_conv_tc|k_conv_out" -s 12 -c 7 -o /tmp/reps/c5 -f \
  python bench.py --steps 1 --warmup 2 --no-cpu-baseline > $O/ncu_c5.log 2>&1
python tools/ncu_summary.py /tmp/reps/c5.ncu-rep > $O/ncu_c5_summary.txt 2>&1
ncu -i /tmp/reps/c5.ncu-rep --page raw --csv > $O/ncu_c5_raw.csv 2>/dev/null
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain_tx|k_cnn_fused|k_rx_combine" \
  -s 3 -c 3 -o /tmp/reps/c2 -f python bench.py --config C2 --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_c2.log 2>&1
python tools/ncu_summary.py /tmp/reps/c2.ncu-rep > $O/ncu_c2_summary.txt 2>&1
ncu -i /tmp/reps/c2.ncu-rep --page raw --csv > $O/ncu_c2_raw.csv 2>/dev/null
echo done > $O/DONE

# Round-end style record run: GPU tests, bench lines for every config, the launch list and
# ncu --set full captures of the top kernels (summarised on the box; the .ncu-rep files are
# removed there to keep gpurun_out small).  usage: bash tools/gpu_full.sh TAG
T=${1:-v5}
set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests_full_$T.log
timeout 600 python bench.py > gpurun_out/bench_${T}_c2.log 2>&1
timeout 300 python bench.py --impl reference > gpurun_out/bench_${T}_reference.log 2>&1
for c in "C1" "C3 --batch 512" "C4 --batch 128" "C5 --batch 32" "P"; do
  tag=$(echo $c | cut -d' ' -f1)
  timeout 400 python bench.py --no-cpu-baseline --config $c > gpurun_out/bench_${T}_$tag.log 2>&1
done
timeout 400 python bench.py --no-cpu-baseline --impair > gpurun_out/bench_${T}_impair.log 2>&1
timeout 400 python bench.py --no-cpu-baseline --redraw --steps 10 > gpurun_out/bench_${T}_redraw.log 2>&1
timeout 400 python bench.py --no-cpu-baseline --unfused > gpurun_out/bench_${T}_unfused.log 2>&1
timeout 600 python tools/stage_bench.py C2 1024 10 > gpurun_out/stage_${T}_c2.json 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_$T.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_$T.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_$T.log 2>&1
mkdir -p /tmp/reps
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain_tx|k_cnn_fused|k_rx_combine" -s 3 -c 3 -o /tmp/reps/c2 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_${T}.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_conv" -s 0 -c 5 -o /tmp/reps/cnn_c5 -f python tools/cnn_one.py C5 64 > gpurun_out/ncu_${T}_cnn.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:"k_chain_cl|k_precode|k_rx_combine" -s 3 -c 3 -o /tmp/reps/c5 -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C5 --batch 32 > gpurun_out/ncu_${T}_c5.log 2>&1
for r in c2 cnn_c5 c5; do
  python tools/ncu_summary.py /tmp/reps/$r.ncu-rep > gpurun_out/ncu_${T}_${r}_summary.txt 2>&1
  ncu -i /tmp/reps/$r.ncu-rep --page raw --csv > gpurun_out/ncu_${T}_${r}_raw.csv 2>/dev/null
done
ncu -i /tmp/reps/c2.ncu-rep --page source --csv --print-source sass -k regex:k_chain_tx 2>/dev/null > /tmp/reps/sass_c2.csv
python tools/sass_stalls.py /tmp/reps/sass_c2.csv > gpurun_out/ncu_${T}_c2_chain_phases.txt 2>&1
python tools/sass_phases.py /tmp/reps/sass_c2.csv >> gpurun_out/ncu_${T}_c2_chain_phases.txt 2>&1

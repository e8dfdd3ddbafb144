timeout 600 python -m pytest tests -m gpu -q -x -k "precode or large" 2>&1 | tail -2 > gpurun_out/tests_pc.log
for c in "C4 --batch 128" "C5 --batch 32"; do
  tag=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 10 --warmup 3 > gpurun_out/bench_pc_$tag.log 2>&1
done
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C5 --batch 32 > /dev/null 2>&1; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c5.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C5 --batch 32 > /dev/null 2>&1

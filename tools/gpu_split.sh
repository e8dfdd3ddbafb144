set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "precode or chain_txrx" 2>&1 | tail -3 > gpurun_out/tests_split.log
for c in "C2" "C2 --split-precode" "C3 --batch 512 --split-precode" "C4 --batch 128 --split-precode" "C5 --batch 32 --split-precode"; do
  tag=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 10 --warmup 3 > gpurun_out/bench_sp_$tag.log 2>&1
done

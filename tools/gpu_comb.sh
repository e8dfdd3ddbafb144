set -x
timeout 600 python -m pytest tests -m gpu -q -x -k "combine or chain_txrx or runtime or dist or shard" 2>&1 | tail -3 > gpurun_out/tests_comb.log
for c in "C2" "C4 --batch 128" "C5 --batch 32"; do
  tag=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 10 --warmup 3 > gpurun_out/bench_cb_$tag.log 2>&1
done

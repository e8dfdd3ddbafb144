timeout 900 python -m pytest tests -m gpu -q -x -k "ofdm or chain or receive or end_to_end or gmp or large" 2>&1 | tail -2 > gpurun_out/tests_tw.log
for c in "C2" "C3 --batch 512" "C5 --batch 32"; do
  tag=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 20 --warmup 3 > gpurun_out/bench_tw_$tag.log 2>&1
done

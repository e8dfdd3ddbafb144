timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tests_cl.log
for c in "C3 --batch 512" "C4 --batch 128" "C5 --batch 32"; do
  tag=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 10 --warmup 3 > gpurun_out/bench_cl_$tag.log 2>&1
done

timeout 900 python -m pytest tests -m gpu -q -x -k "cnn or fdcnn or precode or runtime or end_to_end or e2e" 2>&1 | tail -3 > gpurun_out/tests_cf.log
timeout 300 python tools/cnn_time.py C2:1024 C3:256 C4:256 C5:64 > gpurun_out/cnn_time.log 2>&1
for c in "C2" "C4 --batch 128" "C5 --batch 32"; do
  tag=$(echo $c | tr -d ' -')
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 10 --warmup 3 > gpurun_out/bench_cf_$tag.log 2>&1
done

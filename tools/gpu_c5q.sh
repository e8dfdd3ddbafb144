timeout 900 python -m pytest tests -m gpu -q -x -k "combine or large" 2>&1 | tail -2 > gpurun_out/tests_q.log
timeout 300 python bench.py --no-cpu-baseline --config C5 --batch 32 --steps 10 --warmup 3 > gpurun_out/bench_q5.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --config C4 --batch 128 --steps 10 --warmup 3 > gpurun_out/bench_q4.log 2>&1

timeout 900 python -m pytest tests -m gpu -q -x -k "chain or end_to_end or precode or impair or redraw or runtime" 2>&1 | tail -2 > gpurun_out/tests_q.log
timeout 300 python bench.py --no-cpu-baseline --steps 30 --warmup 3 > gpurun_out/bench_q.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --config C3 --batch 512 --steps 10 --warmup 3 > gpurun_out/bench_q3.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --config P --steps 30 --warmup 3 > gpurun_out/bench_qp.log 2>&1

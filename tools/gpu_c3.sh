timeout 600 python -m pytest tests -m gpu -q -x -k "ofdm or chain or receive or rx or gmp" 2>&1 | tail -3 > gpurun_out/tests_c3.log
timeout 300 python bench.py --no-cpu-baseline --config C3 --batch 512 --steps 10 --warmup 3 > gpurun_out/bench_c3.log 2>&1

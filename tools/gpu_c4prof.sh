set -x
timeout 600 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tests_c4p.log
timeout 300 python bench.py --no-cpu-baseline --config C4 --batch 128 --steps 10 --warmup 3 > gpurun_out/bench_c4p.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --config C5 --batch 32 --steps 10 --warmup 3 > gpurun_out/bench_c5p.log 2>&1
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C4 --batch 16 > gpurun_out/plain_c4.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_tx -s 3 -c 1 -o gpurun_out/prof_c4p -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C4 --batch 16 > gpurun_out/ncu_c4.log 2>&1

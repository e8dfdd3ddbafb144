set -x
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/gpu_tests_full.log
timeout 600 python bench.py > gpurun_out/bench_v4.log 2>&1
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain_v4.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v4.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch_v4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_tx -s 3 -c 1 -o gpurun_out/prof_v4_chain -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_v4.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_conv_tc -s 1 -c 3 -o gpurun_out/prof_v4_conv_c4 -f python tools/cnn_one.py C4 256 > gpurun_out/ncu_v4c.log 2>&1

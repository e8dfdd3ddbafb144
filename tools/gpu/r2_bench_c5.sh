set -x
nproc; python -c "import os;print(len(os.sched_getaffinity(0)))"; grep -m1 "model name" /proc/cpuinfo; nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python bench.py > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo rc=$?
timeout 900 python bench.py --impl reference > gpurun_out/r2_ref_c5.json 2> gpurun_out/r2_ref_c5.err; echo rc=$?
timeout 300 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2_launches_c5.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_chain_cl -s 2 -c 1 -o gpurun_out/r2_chain_c5 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1; echo rc=$?

set -x
for c in "C3 --batch 512" "C4 --batch 128" "C5 --batch 32"; do
  set -- $c
  timeout 300 python bench.py --no-cpu-baseline --config $c --steps 5 --warmup 3 > gpurun_out/bench_big_$1.log 2>&1
done
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C4 --batch 16 > gpurun_out/plain_c4.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_tx -s 3 -c 1 -o gpurun_out/prof_c4chain -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C4 --batch 16 > gpurun_out/ncu_c4.log 2>&1

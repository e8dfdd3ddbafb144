timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C5 --batch 8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_chain_cl -s 3 -c 1 -o /tmp/clp -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --config C5 --batch 8 > gpurun_out/ncu_clp.log 2>&1
python tools/ncu_summary.py /tmp/clp.ncu-rep > gpurun_out/clp_summary.txt 2>&1
ncu -i /tmp/clp.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/clp_sass.csv
python tools/sass_stalls.py /tmp/clp_sass.csv > gpurun_out/clp_phases.txt 2>&1
python tools/sass_phases.py /tmp/clp_sass.csv >> gpurun_out/clp_phases.txt 2>&1
python tools/sass_wavefronts.py /tmp/clp_sass.csv >> gpurun_out/clp_phases.txt 2>&1

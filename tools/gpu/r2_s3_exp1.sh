#!/bin/bash
# C5 A/B: combine path, precode math, batch 64, GMP tap chunking; ncu --set full of the four C5 kernels.
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/e1_base.json 2>&1
$B --combine simt > gpurun_out/e1_csimt.json 2>&1
$B --precode-math fp32tc > gpurun_out/e1_pfp32tc.json 2>&1
$B --precode-math fp32tc --batch 64 > gpurun_out/e1_b64.json 2>&1
$B --precode-math fp32tc --batch 64 --combine simt > gpurun_out/e1_b64_csimt.json 2>&1
FDPD_LIB=build/var/libvar_tap7.so $B --precode-math fp32tc > gpurun_out/e1_tap7.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:k_chain_cl|k_combine_tc|k_precode_tc|k_conv_tc<64, 64" -s 8 -c 4 -o gpurun_out/e1_c5 -f python bench.py --no-cpu-baseline --steps 1 --warmup 3 --precode-math fp32tc > gpurun_out/e1_ncu.log 2>&1

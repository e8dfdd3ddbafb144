#!/bin/bash
# ncu --set full capture of the cluster chain with the tensor-core GMP (after a plain run exits 0)
B="python bench.py --no-cpu-baseline --steps 1 --warmup 3 --gmp ${GMP:-tc}"
timeout 300 $B > gpurun_out/chain_prof_plain.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_chain_cl -s 3 -c 1 \
  --metrics l1tex__data_pipe_tc_wavefronts_mem_shared.sum,sm__inst_executed_pipe_tc.sum,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_tc_wavefronts.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active \
  -o gpurun_out/chain_prof_${GMP:-tc} -f $B > gpurun_out/chain_prof_ncu.log 2>&1

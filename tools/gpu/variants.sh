#!/bin/bash
# A/B of variant builds under variants/: bench C5 with each
B="timeout 300 python bench.py --no-cpu-baseline --steps 10 --warmup 3"
$B > gpurun_out/var_default.json 2>&1
for v in variants/libfdpd_*.so; do
  n=$(basename $v .so)
  FDPD_LIB=$PWD/$v $B > gpurun_out/var_$n.json 2>&1
done

#!/bin/bash
# usage: tools/gpu_prof.sh TAG [ncu-kernel-regex] [bench-args...]
# On the GPU box: full GPU tests, a bench line, and (optional) one ncu --set full
# capture with source of the named kernel from a 64-symbol bench run.
TAG="$1"; NCU="$2"; shift 2; BARGS="$*"
CMD="timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -3 > gpurun_out/tests_$TAG.log; timeout 600 python bench.py --no-cpu-baseline $BARGS > gpurun_out/bench_$TAG.log 2>&1"
if [ -n "$NCU" ]; then
  CMD="$CMD; timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 64 $BARGS > gpurun_out/plain_$TAG.log 2>&1 && timeout 900 ncu --set full --clock-control none --import-source on -k regex:$NCU -s 3 -c 1 -o gpurun_out/prof_$TAG -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 64 $BARGS > gpurun_out/ncu_$TAG.log 2>&1"
fi
timeout 2700 /usr/local/graft/bin/gpurun --timeout 1800 -- "$CMD" 2>&1 | tail -2
cat gpurun_out/tests_$TAG.log
python - "$TAG" <<'PY'
import json, sys
for l in open(f'gpurun_out/bench_{sys.argv[1]}.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()}, 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    else: print(l[:300].rstrip())
PY
if [ -n "$NCU" ] && [ -f gpurun_out/prof_$TAG.ncu-rep ]; then
  python tools/ncu_summary.py gpurun_out/prof_$TAG.ncu-rep
  ncu -i gpurun_out/prof_$TAG.ncu-rep --page source --csv --print-source sass 2>/dev/null > gpurun_out/sass_$TAG.csv; python tools/sass_phases.py gpurun_out/sass_$TAG.csv 2>/dev/null
fi

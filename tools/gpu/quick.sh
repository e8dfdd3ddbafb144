#!/bin/bash
# usage: tools/gpu_quick.sh "<pytest -k expr or empty>" [ncu-kernel-regex]
# GPU tests (subset), a bench line, and optionally one ncu --set full capture of a kernel.
K="$1"; NCU="$2"
CMD="python -m pytest tests -m gpu -q -x ${K:+-k \"$K\"} 2>&1 | tail -3 > gpurun_out/gpu_tests.log; python bench.py --no-cpu-baseline > gpurun_out/bench.log 2>&1"
if [ -n "$NCU" ]; then
  CMD="$CMD; python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 64 > gpurun_out/plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:$NCU -s 3 -c 1 -o gpurun_out/prof_quick -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --batch 64 > gpurun_out/ncu.log 2>&1"
fi
timeout 2700 /usr/local/graft/bin/gpurun --timeout 1800 -- "$CMD" 2>&1 | tail -1
cat gpurun_out/gpu_tests.log
python - <<'PY'
import json
for l in open('gpurun_out/bench.log'):
    if l.startswith('{'):
        d=json.loads(l); print(round(d['value']), round(d['ms_per_step'],3), {k:round(v,3) for k,v in d['stage_ms'].items()}, 'frac', round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks']['sm_mhz'], d['clocks']['reasons'])
    else: print(l[:300].rstrip())
PY
if [ -n "$NCU" ] && [ -f gpurun_out/prof_quick.ncu-rep ]; then
  python tools/ncu_summary.py gpurun_out/prof_quick.ncu-rep
  ncu -i gpurun_out/prof_quick.ncu-rep --page source --csv --print-source sass 2>/dev/null > /tmp/sass.csv; python tools/sass_phases.py /tmp/sass.csv 2>/dev/null
fi

#!/usr/bin/env python
"""Print the stage times of bench.py JSON lines: python tools/benchline.py file..."""
import json, sys
for f in sys.argv[1:]:
    try:
        for l in open(f):
            if l.startswith('{'):
                d = json.loads(l)
                print(f.split('/')[-1], round(d['value']), round(d['ms_per_step'], 3),
                      {k: round(v, 3) for k, v in d['stage_ms'].items() if k != 'zf_build_once_s'},
                      'frac', round(d['roofline']['frac'], 3), 'e2e', round(d['e2e']['value']) if d.get('e2e') else None)
    except Exception as e:
        print(f, 'ERR', e)

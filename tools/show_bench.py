"""Summarise bench.py JSON lines (files or stdin)."""
import json
import sys

srcs = sys.argv[1:] or ["-"]
for f in srcs:
    fh = sys.stdin if f == "-" else open(f)
    for l in fh:
        if not l.startswith('{'):
            continue
        d = json.loads(l)
        print(f, 'ms/step %.2f' % d['ms_per_step'], 'value %.3g' % d['value'],
              'stage_frac %.3f' % d.get('stage_roofline', {}).get('frac', 0))
        print('  ', {k: round(v['ms_per_step'], 2) for k, v in list(d.get('kernels', {}).items())[:12]})
        print('  ', d.get('mst'))

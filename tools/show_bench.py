import sys, json
for f in sys.argv[1:]:
    for l in open(f):
        if not l.startswith('{'): continue
        d = json.loads(l)
        print(f, 'ms/step %.1f' % d['ms_per_step'], 'value %.3g' % d['value'])
        print('  ', {k: round(v['ms_per_step'], 2) for k, v in list(d['kernels'].items())[:10]})
        print('  ', d.get('mst'), 'entries' , d['roofline'] and d['roofline'].get('algo_bytes_per_launch'))

#!/usr/bin/env python
"""Per-launch DRAM bytes of every kernel of the LAST bench step in an ncu metrics
launch list (gpu__time_duration + dram__bytes_read/write, tools/gpu_profile_r02c.sh)
into profiles/ncu_traffic.json -- bench.py's roofline `traffic` field.
usage: python tools/traffic_from_launches.py launches.csv source-label"""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SC = {'byte': 1, 'ns': 1e-6}


def main(path, label):
    rows = list(csv.reader(open(path)))
    st = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    h = rows[st]
    ki, mi, vi, ui, ii = (h.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    per = {}
    for r in rows[st + 1:]:
        d = per.setdefault(int(r[ii]), {'name': r[ki]})
        d[r[mi]] = float(r[vi].replace(',', '')) * SC.get(r[ui], 1.0)
    ids = sorted(per)
    start = max(i for i in ids if 'k_core_mark' in per[i]['name'])
    end = min(i for i in ids if i > start and 'k_label' in per[i]['name'])
    agg = {}
    for i in ids[ids.index(start):ids.index(end) + 1]:
        m = re.search(r'(k_\w+)', per[i]['name'])
        if not m:
            continue
        a = agg.setdefault(m.group(1), [0, 0.0])
        a[0] += 1
        a[1] += per[i].get('dram__bytes_read.sum', 0) + per[i].get('dram__bytes_write.sum', 0)
    out = os.path.join(ROOT, 'profiles', 'ncu_traffic.json')
    cur = json.load(open(out)) if os.path.exists(out) else {}
    for n, (cnt, b) in agg.items():
        cur[n] = {'dram_bytes_per_launch': b / cnt, 'launches_captured': cnt,
                  'source': f'{label} (all {cnt} launches of one C4 step, ncu dram metrics pass)'}
    json.dump(cur, open(out, 'w'), indent=1)
    print(json.dumps({n: round(v['dram_bytes_per_launch'] / 1e9, 3) for n, v in cur.items()}))


if __name__ == '__main__':
    main(sys.argv[1], sys.argv[2])

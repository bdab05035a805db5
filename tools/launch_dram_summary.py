#!/usr/bin/env python
"""Per-kernel time share and DRAM bytes of the LAST bench step in an ncu launch list taken with
--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum (tools/gpu_final_r02s4.sh):
the launches from the last k_core_mark to the k_label after it.
usage: python tools/launch_dram_summary.py launches.csv > profiles/rNN/launches_<tag>_summary.txt"""
import csv
import re
import sys

SC = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-6, 'us': 1e-3, 'ms': 1.0, 's': 1e3,
      'nsecond': 1e-6, 'usecond': 1e-3, 'msecond': 1.0, 'second': 1e3}


def short(name):
    m = re.search(r'(k_[a-z0-9_]+|Device[A-Za-z]+Kernel|Device[A-Za-z]+)', name)
    return m.group(1) if m else name[:40]


def main(path):
    rows = list(csv.reader(l for l in open(path) if l.startswith('"')))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    launches = {}
    for r in rows[1:]:
        d = launches.setdefault(int(r[ii]), {'name': r[ki], 'ms': 0.0, 'bytes': 0.0})
        val = float(r[vi].replace(',', '')) * SC.get(r[ui], 1)
        if 'time_duration' in r[mi]:
            d['ms'] = val
        else:
            d['bytes'] += val
    ids = sorted(launches)
    start = max(i for i in ids if 'k_core_mark' in launches[i]['name'])
    end = min(i for i in ids if i > start and 'k_label' in launches[i]['name'])
    per = {}
    for i in ids:
        if start <= i <= end:
            L = launches[i]
            p = per.setdefault(short(L['name']), [0, 0.0, 0.0])
            p[0] += 1
            p[1] += L['ms']
            p[2] += L['bytes']
    tot = sum(p[1] for p in per.values())
    totb = sum(p[2] for p in per.values())
    print(f"{'kernel':46s} {'launches':>8s} {'ms':>8s} {'share':>7s} {'DRAM GB':>8s} {'GB/s':>7s}")
    for n, p in sorted(per.items(), key=lambda kv: -kv[1][1]):
        print(f"{n:46s} {p[0]:8d} {p[1]:8.3f} {100 * p[1] / tot:6.1f}% {p[2] / 1e9:8.2f} {p[2] / 1e6 / max(p[1], 1e-9):7.0f}")
    print(f"{'total':46s} {sum(p[0] for p in per.values()):8d} {tot:8.3f} {100.0:6.1f}% {totb / 1e9:8.2f}")


if __name__ == '__main__':
    main(sys.argv[1])

#!/usr/bin/env python
"""Per-step DRAM budget from an ncu metrics pass over every kernel of a bench step
(tools/gpu_dram_budget.sh): sum of dram__bytes_read + dram__bytes_write per kernel
name over the LAST step's launches, from its k_core_mark to its k_label (bench.py
runs two steps: un-instrumented and instrumented; the NMI quality pass after them
is not part of a step), against the algorithmic bytes 8 N k + 4 N + N/8.
usage: python tools/dram_budget.py dram_all.csv N k > profiles/r02/dram_budget_c4.txt"""
import csv
import sys

SC = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9}


def main(path, N, k):
    rows = list(csv.reader(open(path)))
    st = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
    hdr = rows[st]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ('Kernel Name', 'Metric Name', 'Metric Value', 'Metric Unit', 'ID'))
    per = {}
    for r in rows[st + 1:]:
        d = per.setdefault(int(r[ii]), {'name': r[ki]})
        d[r[mi]] = float(r[vi].replace(',', '')) * SC.get(r[ui], 1.0)
    ids = sorted(per)
    # the last step starts at the last k_core_mark launch
    start = max(i for i in ids if 'k_core_mark' in per[i]['name'])
    end = min(i for i in ids if i > start and 'k_label' in per[i]['name'])  # the step ends with kdb_label
    agg = {}
    for i in ids:
        if i < start or i > end:
            continue
        d = per[i]
        nm = d['name'].split('(')[0].replace('void ', '').replace('<unnamed>::', '').split('<')[0].strip()[:44]
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += d.get('dram__bytes_read.sum', 0) + d.get('dram__bytes_write.sum', 0)
    tot = sum(v[1] for v in agg.values())
    algo = 8.0 * N * k + 4.0 * N + N / 8.0
    print(f"# DRAM bytes (read + write) per kernel, one C4 step (ncu, cold cache per launch); algorithmic {algo / 1e9:.1f} GB")
    print(f"{'kernel':46s} {'launches':>8s} {'GB':>9s} {'share':>7s}")
    for nm, (n, b) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{nm:46s} {n:8d} {b / 1e9:9.2f} {b / tot * 100:6.1f}%")
    print(f"{'total':46s} {sum(v[0] for v in agg.values()):8d} {tot / 1e9:9.2f}   ratio to algorithmic {tot / algo:.2f}")


if __name__ == '__main__':
    main(sys.argv[1], int(sys.argv[2]), int(sys.argv[3]))

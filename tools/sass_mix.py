#!/usr/bin/env python
"""Opcode mix of one kernel from an `ncu --page source --csv --print-source sass` export
(tools/gpu_final_r02s4.sh: source_lr_<tag>.csv): share of executed warp instructions, share of
stall samples and average active lanes per opcode, and the same along the program in blocks of 40 SASS lines.
usage: python tools/sass_mix.py source.csv > profiles/rNN/<kernel>_sass_mix.txt"""
import csv
import re
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ia, ie, it, isamp = (hdr.index(x) for x in ('Source', 'Instructions Executed', 'Thread Instructions Executed', '# Samples'))
ins = []
for r in rows[2:]:
    try:
        ins.append((r[ia].strip(), int(r[ie]), int(r[it]), int(r[isamp])))
    except (ValueError, IndexError):
        pass
tot, tots = sum(x[1] for x in ins), sum(x[3] for x in ins)
print(f"# {rows[0][1][:90]}...")
print(f"# {len(ins)} SASS instructions, {tot:.3e} warp instructions executed, {tots} stall samples")
c, cs, ct = Counter(), Counter(), Counter()
for s_, e, t, sm in ins:
    op = re.sub(r'^@!?U?P\d+\s+', '', s_).split()[0].split('.')[0]
    c[op] += e
    cs[op] += sm
    ct[op] += t
print(f"{'opcode':10s} {'inst %':>7s} {'samples %':>10s} {'lanes':>6s}")
for op, e in c.most_common(24):
    print(f"{op:10s} {100 * e / tot:7.1f} {100 * cs[op] / tots:10.1f} {ct[op] / max(e, 1):6.1f}")
print("# along the program, 40 SASS lines per block: first line index, share of executed instructions, active lanes")
for i in range(0, len(ins), 40):
    seg = ins[i:i + 40]
    e = sum(x[1] for x in seg)
    if e * 200 >= tot:
        print(f"{i:5d} {100 * e / tot:5.1f}% lanes {sum(x[2] for x in seg) / max(1, e):4.1f}")

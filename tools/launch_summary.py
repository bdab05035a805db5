"""Per-kernel totals of ONE bench step from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --csv --log-file X.csv python bench.py --steps 1 ...`).
The step is the launches from the first k_core_mark up to the next one.
usage: python tools/launch_summary.py launches.csv > summary.txt"""
import csv
import sys
from collections import OrderedDict


def base(name):
    n = name.replace("void ", "").replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    if n.startswith("cub::") or n.startswith("CUB_"):
        return n.split("(")[0][:60]
    return n.split("(")[0].split("<")[0].strip()


rows = [r for r in csv.reader(l for l in open(sys.argv[1]) if l.startswith('"'))]
hdr = rows[0]
K, V = hdr.index("Kernel Name"), hdr.index("Metric Value")
launches = [(base(r[K]), float(r[V].replace(",", ""))) for r in rows[1:]]
starts = [i for i, (n, _) in enumerate(launches) if n == "k_core_mark"]
seg = launches[starts[0]:starts[1]] if len(starts) > 1 else launches[starts[0]:]
tot = OrderedDict()
for n, ns in seg:
    c, t = tot.get(n, (0, 0.0))
    tot[n] = (c + 1, t + ns)
all_ns = sum(t for _, t in tot.values())
print("# ncu --metrics gpu__time_duration.sum --clock-control none, one bench step (C4), per-kernel totals")
print("# (cold-cache, serialised launches: compare SHARES, not absolutes)")
print(f"{'kernel':62s} {'launches':>8s} {'us':>10s} {'share':>7s}")
for n, (c, t) in sorted(tot.items(), key=lambda kv: -kv[1][1]):
    print(f"{n[:62]:62s} {c:8d} {t / 1e3:10.1f} {100 * t / all_ns:6.1f}%")
print(f"{'total':62s} {len(seg):8d} {all_ns / 1e3:10.1f}")

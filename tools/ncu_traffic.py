"""Write profiles/ncu_traffic.json (per-launch DRAM bytes per kernel, averaged
over the captured launches) and a readable summary from an ncu --set full report.
usage: python tools/ncu_traffic.py <summary.txt> <report.ncu-rep | raw.csv> [...]"""
import csv
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'lts__t_sector_hit_rate.pct', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'smsp__inst_executed.sum', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'lts__t_sectors_srcunit_tex_op_read.sum', 'lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum']


def main(out, reps):
  agg, lines, srcs = {}, [], {}
  for rep in reps:
    if rep.endswith('.csv'):  # a raw page already exported on the GPU box (ncu -i rep --page raw --csv)
        raw = open(rep).read()
    else:
        raw = subprocess.run(['ncu', '-i', rep, '--page', 'raw', '--csv'], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        name = r[hdr.index('Kernel Name')]
        base = name.split('(')[0].replace('void ', '').replace('<unnamed>::', '').split('<')[0].strip()
        vals = {}
        for k in KEYS:
            if k in hdr:
                v = r[hdr.index(k)].replace(',', '')
                try:
                    vals[k] = float(v)
                except ValueError:
                    pass
                u = units[hdr.index(k)]
                vals[k + ' [' + u + ']'] = vals.get(k)
        scale = {'Gbyte': 1e9, 'Mbyte': 1e6, 'Kbyte': 1e3, 'byte': 1.0}
        def b(k):
            u = units[hdr.index(k)]
            return vals.get(k, 0.0) * scale.get(u, 1.0)
        tb = b('dram__bytes_read.sum') + b('dram__bytes_write.sum')
        a = agg.setdefault(base, {'launches': 0, 'dram_bytes': 0.0})
        a['launches'] += 1
        a['dram_bytes'] += tb
        srcs[base] = os.path.basename(rep)
        lines.append(f'--- {name[:110]}')
        for k in KEYS:
            if k in hdr:
                lines.append(f'    {k} [{units[hdr.index(k)]}] = {r[hdr.index(k)]}')
  traffic = {k: {'dram_bytes_per_launch': v['dram_bytes'] / v['launches'], 'launches_captured': v['launches'],
                 'source': srcs[k]} for k, v in agg.items()}
  with open(os.path.join(ROOT, 'profiles', 'ncu_traffic.json'), 'w') as f:
    json.dump(traffic, f, indent=1)
  with open(out, 'w') as f:
    f.write(f'# ncu --set full --clock-control none, {", ".join(os.path.basename(r) for r in reps)} (B200, gpurun box)\n')
    f.write('\n'.join(lines) + '\n')
  print(json.dumps(traffic, indent=1))


if __name__ == '__main__':
  main(sys.argv[1], sys.argv[2:])

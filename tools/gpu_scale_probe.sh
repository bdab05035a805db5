#!/bin/bash
# Per-record cost of the light rounds against cluster size (working-set probe).
mkdir -p gpurun_out
for s in 0.125 0.25 0.5 1.0; do
  KDB_TRACE=1 python bench.py --config C4 --scale $s --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/sp_$s.json 2> gpurun_out/sp_$s.err
  python - "$s" <<'PY'
import json, re, sys
s = sys.argv[1]
d = json.loads(open(f"gpurun_out/sp_{s}.json").read().strip().splitlines()[-1])
lr = sum(v["ms_per_step"] for k, v in d["kernels"].items() if "k_light_round" in k)
lines = [l for l in open(f"gpurun_out/sp_{s}.err") if l.startswith("[kdb] round")]
nr = len(lines) // 3  # warmup + timed + instrumented steps
live = sum(int(re.search(r"live=(\d+)", l).group(1)) for l in lines[:nr])
print(f"scale {s}: N={d['config']['N']} ms/step {d['ms_per_step']:.2f} light_round {lr:.2f} ms records {live} "
      f"-> {lr * 1e9 / max(live, 1):.1f} ps/record")
PY
done

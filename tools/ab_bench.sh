#!/bin/bash
# A/B timing of library variants on one config: each line = one bench run.
# usage: tools/ab_bench.sh <tag> <config> "<ENV=.. label>" ...
TAG=$1; CFG=$2; shift 2
mkdir -p gpurun_out
for v in "$@"; do
  env $v python bench.py --config $CFG --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ab_${TAG}.tmp 2> gpurun_out/ab_${TAG}.err
  echo "== $v rc=$?"
  tail -1 gpurun_out/ab_${TAG}.tmp | tee -a gpurun_out/ab_${TAG}.jsonl | python tools/show_bench.py 2>/dev/null | head -30
done

#!/bin/bash
# One gpurun call: full-size window parity of the benchmarked path (C4, C5 x1/4)
# and the whole-workload oracle timing; logs under gpurun_out/.
set -u
mkdir -p gpurun_out
python tools/window_parity.py --config C4 --scale 0.01 --workers 4 --out gpurun_out/wp_C4_small.json \
    > gpurun_out/wp_C4_small.log 2>&1; echo "small rc=$?"
tail -3 gpurun_out/wp_C4_small.log
python tools/window_parity.py --config C4 --workers ${W:-5} --out gpurun_out/window_parity_C4.json \
    --golden gpurun_out/window_oracle_C4.json > gpurun_out/wp_C4.log 2>&1; echo "C4 rc=$?"
tail -14 gpurun_out/wp_C4.log | cut -c1-400
python tools/window_parity.py --config C5 --scale 0.25 --workers ${W:-5} --out gpurun_out/window_parity_C5q.json \
    --golden gpurun_out/window_oracle_C5q.json > gpurun_out/wp_C5q.log 2>&1; echo "C5q rc=$?"
tail -14 gpurun_out/wp_C5q.log | cut -c1-400

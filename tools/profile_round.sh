#!/bin/bash
# One gpurun call: full bench line, ncu launch list, one --set full capture.
# usage: tools/profile_round.sh <tag> <kernel-regex> <skip>
set -u
TAG=${1:-r01}; KRE=${2:-k_offer_rows_t}; SKIP=${3:-6}
mkdir -p gpurun_out
python bench.py --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?"
ARGS="--steps 1 --warmup 1 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches_${TAG}.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:${KRE} -s ${SKIP} -c 1 \
    -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu rc=$?"

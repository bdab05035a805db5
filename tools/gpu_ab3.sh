# A/B on one box: evict-last hint on the light-round component gathers (KDB_L2HINT)
mkdir -p gpurun_out
ARGS="--steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
: > gpurun_out/ab3.jsonl
for rep in 1 2; do for h in 0 1; do KDB_L2HINT=$h timeout 300 python bench.py $ARGS 2>/dev/null | tail -1 >> gpurun_out/ab3.jsonl; done; done
KDB_L2HINT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c1 or random or points" > gpurun_out/ab3_tests.log 2>&1; echo "tests rc=$?"

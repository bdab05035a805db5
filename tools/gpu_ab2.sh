# A/B on one box: round-2 head skip (KDB_SKIP1) on C4; two-level global phase (KDB_GMAP) under sim 8
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_first.py -x -q > gpurun_out/ab2_tests.log 2>&1; echo "tests rc=$?"
ARGS="--steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
: > gpurun_out/ab2.jsonl
for rep in 1 2; do
for s in 0 1; do KDB_SKIP1=$s timeout 300 python bench.py $ARGS 2>/dev/null | tail -1 >> gpurun_out/ab2.jsonl; done
done
for g in 0 1; do KDB_GMAP=$g timeout 600 python bench.py $ARGS --sim 8 2>/dev/null | tail -1 >> gpurun_out/ab2.jsonl; done
echo done

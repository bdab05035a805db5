# per-lane state-machine light rounds (KDB_LRSM): parity, then A/B on one box
mkdir -p gpurun_out
KDB_LRSM=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_first.py tests/test_gpu_edge_cols.py -x -q > gpurun_out/ab4_tests.log 2>&1; echo "tests rc=$?"
ARGS="--steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
: > gpurun_out/ab4.jsonl
for rep in 1 2; do for h in 0 1; do KDB_LRSM=$h timeout 300 python bench.py $ARGS 2>/dev/null | tail -1 >> gpurun_out/ab4.jsonl; done; done
for c in C3 C2; do for h in 0 1; do KDB_LRSM=$h timeout 300 python bench.py --config $c $ARGS 2>/dev/null | tail -1 >> gpurun_out/ab4.jsonl; done; done
echo done

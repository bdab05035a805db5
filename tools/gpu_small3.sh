# fused contraction bookkeeping: parity (parity, local-first, configs C2/C3, debug build) + C1..C4 lines
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_first.py tests/test_gpu_debug.py tests/test_gpu_configs.py -x -q -k "not c4 and not c5" > gpurun_out/small3_tests.log 2>&1; echo "tests rc=$?"
ARGS="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
: > gpurun_out/small3.jsonl
for c in C1 C2 C3 C4; do timeout 300 python bench.py --config $c $ARGS 2>/dev/null | tail -1 >> gpurun_out/small3.jsonl; done
echo done

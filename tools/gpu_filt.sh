mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -k "filter" -x -q > gpurun_out/filt_tests.log 2>&1; echo "tests rc=$?"
ARGS="--steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
: > gpurun_out/filt_bench.jsonl
timeout 300 python bench.py $ARGS --out gpurun_out/filt_bench.jsonl > /dev/null 2>&1; echo "bench rc=$?"
timeout 300 python bench.py $ARGS --edge-cols M --out gpurun_out/filt_bench.jsonl > /dev/null 2>&1; echo "bench ecM rc=$?"
bash tools/gpu_dram_budget.sh

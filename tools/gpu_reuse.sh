# eps sweep with the kept light ELL: reuse tests + parity subset + sweep bench with/without reuse
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_eps_reuse.py tests/test_gpu_parity.py tests/test_eps_properties.py -x -q > gpurun_out/reuse_tests.log 2>&1; echo "tests rc=$?"
ARGS="--steps 3 --warmup 2 --no-e2e --no-cpu-baseline --eps-factors 0.5,1,1.5,2"
: > gpurun_out/reuse.jsonl
for r in 1 0; do KDB_REUSE=$r timeout 600 python bench.py $ARGS 2>/dev/null | tail -1 >> gpurun_out/reuse.jsonl; done
timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 >> gpurun_out/reuse.jsonl
echo done

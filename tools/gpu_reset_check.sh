# round-start counter reset in one launch: parity, then small configs and C4
mkdir -p gpurun_out
TAG=${1:-rs}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_first.py tests/test_gpu_eps_reuse.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for c in C1 C1 C2 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_$c.log 2>&1; echo "$c rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_$c.log | head -1)"; done

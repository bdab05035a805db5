# L1-cached component gathers (auto on spatially ordered ids): parity, then same-box A/B in both orders
mkdir -p gpurun_out
TAG=${1:-l1}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_local_first.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for rep in 1 2; do for o in inertial generation; do for l in -1 0; do
KDB_L1GAT=$l timeout 900 python bench.py --order $o --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_${o}_$l.log 2>&1; echo "$o l1=$l rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_${o}_$l.log | head -1)"
done; done; done

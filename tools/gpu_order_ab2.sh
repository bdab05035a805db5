# parity of the changed kernels, then the order A/B on C4
mkdir -p gpurun_out
TAG=${1:-ordb}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 3 gpurun_out/parity_${TAG}.log
for o in ${ORDERS:-generation inertial}; do
timeout 1500 python bench.py --config ${CFG:-C4} --order $o --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_${o}.log 2>&1; echo "$o rc=$?"
grep -o '"order": "[^"]*"' gpurun_out/bench_${TAG}_${o}.log
done

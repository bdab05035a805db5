# counting-sort finalize: parity (incl. hub / star forests), C4 bench A/B (radix vs counting), sim scaling lines
mkdir -p gpurun_out
TAG=${1:-ms}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_local_first.py tests/test_gpu_debug.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for v in 1 0 1 0; do KDB_MSF_COUNT=$v timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_${TAG}_count$v.jsonl > gpurun_out/bench_${TAG}_count$v.log 2>&1; echo "count=$v rc=$?"; done
for P in 2 4 8; do timeout 900 python bench.py --sim $P --no-cpu-baseline --no-e2e --steps 3 --out gpurun_out/${TAG}_sim.jsonl > gpurun_out/${TAG}_sim$P.log 2>&1; echo "sim $P rc=$?"; done

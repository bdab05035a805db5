# tile round (kdb_tile.cuh): parity suite, then C4 with tile on/off in both point orders
mkdir -p gpurun_out
TAG=${1:-tile}
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge_cols.py tests/test_gpu_eps_reuse.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 5 gpurun_out/parity_${TAG}.log
for o in ${ORDERS:-inertial generation}; do for t in ${TILES:-1 0}; do
KDB_TILE=$t timeout 900 python bench.py --config ${CFG:-C4} --order $o --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_${o}_$t.log 2>&1; echo "$o tile=$t rc=$?"
done; done
KDB_TRACE=1 timeout 900 python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"

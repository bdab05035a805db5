# tile round iteration: parity (short), bench inertial tile on/off, trace, ncu of k_tile_round
mkdir -p gpurun_out
TAG=${1:-tile}
KDB_TILE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for t in ${TILES:-1 0}; do
KDB_TILE=$t timeout 900 python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_$t.log 2>&1; echo "tile=$t rc=$?"
done
KDB_TILE=1 KDB_TRACE=1 timeout 900 python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"
KDB_TILE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_round -c 1 -o gpurun_out/${TAG}_ncu python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 0 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"

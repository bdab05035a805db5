# tile round variants: parity with the tile on, then (rows per tile, max in-tile rounds) on C4 inertial
mkdir -p gpurun_out
TAG=${1:-tile}
KDB_TILE=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
KDB_TILE=1 KDB_TILE_ROWS=512 timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "random or torus or fuzz" > gpurun_out/parity512_${TAG}.log 2>&1; echo "parity512 rc=$?"; tail -n 2 gpurun_out/parity512_${TAG}.log
for v in ${VARIANTS:-"1 1024 48" "1 1024 3" "1 512 48" "1 512 3" "0 1024 48"}; do
set -- $v
KDB_TILE=$1 KDB_TILE_ROWS=$2 KDB_TILE_MAXR=$3 timeout 900 python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_$1_$2_$3.log 2>&1; echo "tile=$1 rows=$2 maxr=$3 rc=$?"
done
KDB_TILE=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_tile_round -c 1 -o gpurun_out/${TAG}_ncu python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 0 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"

# ELL planes: parity suite, then C4 both orders (+ L1-cached gathers), C1-C3 both orders
mkdir -p gpurun_out
TAG=${1:-pl}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge_cols.py tests/test_gpu_eps_reuse.py tests/test_gpu_local_first.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for v in "C4 inertial 0" "C4 inertial 1" "C4 generation 0" "C3 inertial 0" "C3 generation 0" "C2 inertial 0" "C2 generation 0" "C1 inertial 0" "C1 generation 0"; do
set -- $v
KDB_L1GAT=$3 timeout 900 python bench.py --config $1 --order $2 --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_$1_$2_$3.log 2>&1; echo "$1 $2 l1=$3 rc=$?"
done
timeout 900 ncu --set full --clock-control none -k regex:k_light_round -c 1 -o gpurun_out/${TAG}_lr_ncu python bench.py --no-cpu-baseline --no-e2e --steps 1 --warmup 0 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"

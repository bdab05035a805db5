# quick GPU check after a kernel change: main parity tests, one C4 window, bench line
mkdir -p gpurun_out
TAG=${1:-q}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cols.py tests/test_eps_properties.py -m gpu -x -q > gpurun_out/quick_${TAG}.log 2>&1; echo "parity rc=$?"
timeout 600 python bench.py --no-cpu-baseline --no-e2e --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"

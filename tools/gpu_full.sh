# the whole GPU suite + smoke + default bench line
mkdir -p gpurun_out
TAG=${1:-full}
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/gputest_${TAG}.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"

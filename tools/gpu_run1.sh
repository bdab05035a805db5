set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_a.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_a.log
KDB_TRACE=1 timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_trace_a.log 2>&1; echo "bench rc=$?"
tail -40 gpurun_out/bench_trace_a.log

set -x
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_b.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu_b.log
for L in 4 8 12 16; do
KDB_LIGHT=$L KDB_TRACE=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1; echo "bench L=$L rc=$?"
tail -1 gpurun_out/bench_L$L.log | python tools/show_bench.py 2>/dev/null || tail -c 3000 gpurun_out/bench_L$L.log
done

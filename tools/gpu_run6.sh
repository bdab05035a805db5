timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_e.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_e.log
for L in 6 8 10 12; do
KDB_LIGHT=$L timeout 900 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1; echo "bench L=$L rc=$?"
tail -1 gpurun_out/bench_L$L.log | python tools/show_bench.py
done

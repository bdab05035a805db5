timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_c.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_gpu_c.log
for L in 10 16; do
KDB_LIGHT=$L KDB_TRACE=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1; echo "bench L=$L rc=$?"
grep "\[kdb\]" gpurun_out/bench_L$L.log | tail -14
tail -1 gpurun_out/bench_L$L.log | python tools/show_bench.py
done

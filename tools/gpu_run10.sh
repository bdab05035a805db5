for L in 8 9 10; do
KDB_LIGHT=$L timeout 900 python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_L$L.log 2>&1; echo "bench L=$L rc=$?"
tail -1 gpurun_out/bench_L$L.log | python tools/show_bench.py
done

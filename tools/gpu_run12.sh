timeout 900 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_e.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_e.log | python tools/show_bench.py

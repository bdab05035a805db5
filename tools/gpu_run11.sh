timeout 900 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_e.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_e.log | python tools/show_bench.py
tail -1 gpurun_out/bench_e.log | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['roofline'])"
for C in C3; do
timeout 900 python bench.py --config $C --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1; echo "bench $C rc=$?"
tail -1 gpurun_out/bench_$C.log | python tools/show_bench.py
done

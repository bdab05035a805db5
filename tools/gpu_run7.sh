timeout 900 python -m pytest tests/test_gpu_knng.py -x -q > gpurun_out/pytest_knng.log 2>&1; echo "pytest knng rc=$?"; tail -5 gpurun_out/pytest_knng.log
for C in C2 C3; do
timeout 1200 python bench.py --config $C --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_$C.log 2>&1; echo "bench $C rc=$?"
tail -1 gpurun_out/bench_$C.log | python tools/show_bench.py; grep graph_build gpurun_out/bench_$C.log | head -1 | python -c "import sys,json; d=json.loads(sys.stdin.read()); print(d['config'])"
done

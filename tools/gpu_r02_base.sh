# round-2 baseline: GPU test suite, bench line, ncu launch list (one gpurun call)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r02.log 2>&1; echo "pytest rc=$?"
timeout 600 python bench.py --out gpurun_out/bench_r02.jsonl > gpurun_out/bench_r02.log 2>&1; echo "bench rc=$?"
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r02.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches_r02.log 2>&1; echo "ncu rc=$?"

# full GPU suite + default bench line + per-config lines (current defaults)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_r02b.log 2>&1; echo "gpu tests rc=$?"; tail -n 3 gpurun_out/gputest_r02b.log
timeout 900 python bench.py --out gpurun_out/bench_r02b.jsonl > gpurun_out/bench_r02b.log 2>&1; echo "bench rc=$?"
for c in C1 C2 C3; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_r02b_configs.jsonl > gpurun_out/bench_r02b_$c.log 2>&1; echo "$c rc=$?"; done

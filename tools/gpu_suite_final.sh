# whole GPU suite with the final code, smoke, then bench lines (C1, C4)
mkdir -p gpurun_out
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_final.log 2>&1; echo "gpu tests rc=$?"; tail -n 3 gpurun_out/gputest_final.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_final.log 2>&1; echo "smoke rc=$?"; tail -n 2 gpurun_out/smoke_final.log
for c in C1 C4; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_sf.jsonl > gpurun_out/bench_sf_$c.log 2>&1; echo "$c rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_sf_$c.log | head -1)"; done

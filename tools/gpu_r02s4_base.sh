# session 4 of round 2: baseline on this session's build (parity subset, C4 + C1 bench lines)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/s4_parity.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/s4_parity.log
for c in C4 C1; do timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/s4_base.jsonl > gpurun_out/s4_base_$c.log 2>&1; echo "$c rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/s4_base_$c.log | head -1)"; done

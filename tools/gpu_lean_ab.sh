# scan_ell_lean: parity (tie-heavy suites), then same-box A/B on C4 (both orders) and C3
mkdir -p gpurun_out
TAG=${1:-ln}
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_edge_cols.py tests/test_gpu_eps_reuse.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for rep in 1 2; do for l in 1 0; do
KDB_LEAN=$l timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_$l.log 2>&1; echo "C4 lean=$l rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_$l.log | head -1)"
done; done
for l in 1 0; do KDB_LEAN=$l timeout 900 python bench.py --order generation --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/bench_${TAG}_gen_$l.log 2>&1; echo "C4gen lean=$l $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_gen_$l.log | head -1)"; done

# session 5: the quad-per-row light round (KDB_QUAD, default on) -- parity first, then a same-box A/B on C4 and C3
mkdir -p gpurun_out
TAG=${1:-quad}
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/quick_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/quick_${TAG}.log
bash tools/gpu_ab_multi.sh ab_${TAG} "KDB_QUAD=0" "KDB_QUAD=1"
for q in 0 1; do KDB_QUAD=$q timeout 600 python bench.py --config C3 --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/ab_${TAG}_c3.jsonl > gpurun_out/ab_${TAG}_c3_$q.log 2>&1; echo "C3 quad=$q rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}_c3_$q.log | head -1)"; done
timeout 1200 python -m pytest tests/test_gpu_windows.py -m gpu -x -q > gpurun_out/windows_${TAG}.log 2>&1; echo "windows rc=$?"; tail -n 2 gpurun_out/windows_${TAG}.log

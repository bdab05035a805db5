# session 5: level-synchronous light round (KDB_LVL) -- parity of the kept-off variants, then same-box A/Bs
mkdir -p gpurun_out
TAG=${1:-lvl}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or points_filter or c1_filter" > gpurun_out/quick_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/quick_${TAG}.log
bash tools/gpu_ab_multi.sh ab_${TAG} "KDB_LVL=0" "KDB_LVL=1"
for c in C3 "C5 --scale 0.25"; do for q in 0 1; do KDB_LVL=$q timeout 600 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/ab_${TAG}_cfg.jsonl > gpurun_out/ab_${TAG}_cfg.log 2>&1; echo "$c lvl=$q rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/ab_${TAG}_cfg.log | head -1)"; done; done
KDB_LVL=1 timeout 1200 python -m pytest tests/test_gpu_windows.py -m gpu -x -q > gpurun_out/windows_${TAG}.log 2>&1; echo "windows rc=$?"; tail -n 2 gpurun_out/windows_${TAG}.log

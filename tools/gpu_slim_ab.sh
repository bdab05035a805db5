# session 5: slim builds of the light-round hot loop (libkdb_slim<n>.so, -DKDB_SLIM=n): parity, then same-box A/B on C4
mkdir -p gpurun_out
L=$PWD/paper_2009_04552_b200/lib
for n in "$@"; do
KDB_LIBRARY=$L/libkdb_slim$n.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or points_filter or c1_filter or random_graphs_filter" > gpurun_out/quick_slim$n.log 2>&1; echo "slim$n parity rc=$?"; tail -n 1 gpurun_out/quick_slim$n.log
done
ARGS="KDB_LVL=0"; for n in "$@"; do ARGS="$ARGS KDB_LIBRARY=$L/libkdb_slim$n.so"; done
bash tools/gpu_ab_multi.sh ab_slim $ARGS

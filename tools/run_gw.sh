set -x
python -m pytest tests/test_gpu_edge_cols.py -x -q 2>&1 | tail -2
for gw in 1 2; do KDB_GW=$gw python -m pytest tests/test_gpu_parity.py -x -q -k "random or c1 or points" 2>&1 | tail -2; done
for gw in 4 2 1; do KDB_GW=$gw python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_gw$gw.json 2> gpurun_out/b_gw$gw.err; tail -c 200 gpurun_out/b_gw$gw.err; done
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --edge-cols M > gpurun_out/b_ecM.json 2> gpurun_out/b_ecM.err; tail -c 200 gpurun_out/b_ecM.err

python -m pytest tests/test_gpu_parity.py tests/test_gpu_edge_cols.py -q -x 2>&1 | tail -2
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_f.json 2> gpurun_out/b_f.err; tail -c 300 gpurun_out/b_f.err
python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --edge-cols M > gpurun_out/b_fM.json 2> gpurun_out/b_fM.err; tail -c 300 gpurun_out/b_fM.err

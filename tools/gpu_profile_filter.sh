# One gpurun call: NMI/edge_cols GPU tests + smoke + bench line, then ncu --set full of k_filter and k_label.
mkdir -p gpurun_out
python -m pytest tests/test_nmi.py tests/test_gpu_edge_cols.py -q -x 2>&1 | tail -2
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
python bench.py --out gpurun_out/bench_r01c.jsonl > gpurun_out/bench_r01c.log 2>&1; echo "bench rc=$?"
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_label" -s 0 -c 2 \
    -o gpurun_out/prof_r01c python bench.py $ARGS > gpurun_out/ncu_full_r01c.log 2>&1
echo "ncu full rc=$?"

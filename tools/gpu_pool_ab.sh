# session 5: pooled level scan (KDB_LVL=2) -- parity of the variants, then a same-box A/B on C4
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants" > gpurun_out/quick_pool.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/quick_pool.log
bash tools/gpu_ab_multi.sh ab_pool "KDB_LVL=0" "KDB_LVL=3"
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
KDB_LVL=3 timeout 900 ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum --clock-control none --csv -k regex:"k_light_(round|lvl|pool)" \
    --log-file gpurun_out/lvl_rounds_3.csv python bench.py $ARGS > gpurun_out/lvl_rounds_3.log 2>&1; echo "ncu lvl=3 rc=$?"

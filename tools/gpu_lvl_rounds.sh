# per-round durations of the light-round kernel, default against KDB_LVL=1 (ncu launch list, one C4 step)
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
for q in 0 1; do
  KDB_LVL=$q timeout 900 ncu --metrics gpu__time_duration.sum,smsp__thread_inst_executed_per_inst_executed.ratio,smsp__inst_executed.sum --clock-control none --csv -k regex:"k_light_(round|lvl)" \
    --log-file gpurun_out/lvl_rounds_$q.csv python bench.py $ARGS > gpurun_out/lvl_rounds_$q.log 2>&1; echo "lvl=$q rc=$?"
done

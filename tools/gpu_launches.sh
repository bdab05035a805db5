ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_l.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py $ARGS > gpurun_out/ncu_l.log 2>&1
echo "ncu rc=$?"

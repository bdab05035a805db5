# light round (round 3 = second k_light_round launch): ncu --set full with source, per-line CSV pages; per-round trace
mkdir -p gpurun_out
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
KDB_TRACE=1 timeout 600 python bench.py $ARGS > gpurun_out/trace_c4.log 2>&1; echo "trace rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_light_round -s 1 -c 1 \
    -o /tmp/prof_lr3 python bench.py $ARGS > gpurun_out/ncu_lr3.log 2>&1; echo "ncu rc=$?"
ncu -i /tmp/prof_lr3.ncu-rep --page source --csv --print-source cuda > gpurun_out/source_lr3_cuda.csv 2>&1
ncu -i /tmp/prof_lr3.ncu-rep --page source --csv --print-source sass > gpurun_out/source_lr3_sass.csv 2>&1
ncu -i /tmp/prof_lr3.ncu-rep --page raw --csv > gpurun_out/raw_lr3.csv 2>&1
ls -la gpurun_out; du -sh gpurun_out

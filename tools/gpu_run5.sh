timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_d.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu_d.log
KDB_TRACE=1 timeout 900 python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_d.log 2>&1; echo "bench rc=$?"
grep "\[kdb\]" gpurun_out/bench_d.log | tail -13
tail -1 gpurun_out/bench_d.log | python tools/show_bench.py
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_d.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_light_round -s 0 -c 2 -o gpurun_out/prof_round python bench.py $ARGS > gpurun_out/ncu_round.log 2>&1
echo "ncu1 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_light_ell" -s 0 -c 2 -o gpurun_out/prof_filter python bench.py $ARGS > gpurun_out/ncu_filter.log 2>&1
echo "ncu2 rc=$?"

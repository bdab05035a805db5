# One gpurun call: full bench line (default flags), ncu launch list, ncu --set full of the top kernels.
TAG=${1:-r01}
mkdir -p gpurun_out
python bench.py --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}.log 2>&1
echo "bench rc=$?"
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches_${TAG}.log 2>&1
echo "ncu launches rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_core_mark|k_light_ell|k_light_round|k_hook" -s 0 -c 5 \
    -o gpurun_out/prof_${TAG} python bench.py $ARGS > gpurun_out/ncu_full_${TAG}.log 2>&1
echo "ncu full rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_label|k_relabel|k_tie" -s 0 -c 4 \
    -o gpurun_out/prof2_${TAG} python bench.py $ARGS > gpurun_out/ncu_full2_${TAG}.log 2>&1
echo "ncu full2 rc=$?"
# part B (the light rounds, filter, label): tools/gpu_profile_round_b.sh -- separate call (64 MiB copy-back cap)

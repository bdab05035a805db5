TAG=${1:-r01}
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_light_round" -s 0 -c 13 \
    -o gpurun_out/prof3_${TAG} python bench.py $ARGS > gpurun_out/ncu_full3_${TAG}.log 2>&1
echo "ncu full3 rc=$?"
ncu --set full --clock-control none --import-source on -k regex:"k_filter|k_label" -s 0 -c 2 \
    -o gpurun_out/prof4_${TAG} python bench.py $ARGS > gpurun_out/ncu_full4_${TAG}.log 2>&1
echo "ncu full4 rc=$?"

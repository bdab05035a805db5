# round-2 (session 3) profile of the default path (inertial order): bench line, launch list of
# the repo's kernels, ncu --set full of the top kernels, per-kernel DRAM bytes of one step
TAG=${1:-r02c}
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
timeout 600 python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1; echo "plain rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"k_|cub|Radix|Scan|Select" --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
cap() {  # name regex count
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 0 -c $3 \
      -o /tmp/prof_$1_${TAG} python bench.py $ARGS > gpurun_out/ncu_$1_${TAG}.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i /tmp/prof_$1_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_$1_${TAG}.csv 2>/dev/null
  ncu -i /tmp/prof_$1_${TAG}.ncu-rep --page details --csv > gpurun_out/details_$1_${TAG}.csv 2>/dev/null
}
cap lr "k_light_round" 4
cap st "k_filter|k_light_ell|k_core_mark|k_label" 4
du -sh gpurun_out

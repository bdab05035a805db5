# round-2 profile: bench line, launch list, ncu --set full of the top kernels (one gpurun call).
# The .ncu-rep files are reduced to CSV pages on the box (gpurun copies back <= 64 MiB).
TAG=${1:-r02}
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
mkdir -p gpurun_out
timeout 600 python bench.py --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}.log 2>&1; echo "bench rc=$?"
timeout 600 python bench.py $ARGS > gpurun_out/plain_${TAG}.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${TAG}.csv \
    python bench.py $ARGS > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
cap() {  # name regex count
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"$2" -s 0 -c $3 \
      -o /tmp/prof_$1_${TAG} python bench.py $ARGS > gpurun_out/ncu_$1_${TAG}.log 2>&1; echo "ncu $1 rc=$?"
  ncu -i /tmp/prof_$1_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_$1_${TAG}.csv 2>/dev/null
  ncu -i /tmp/prof_$1_${TAG}.ncu-rep --page details --csv > gpurun_out/details_$1_${TAG}.csv 2>/dev/null
}
cap lr "k_light_round" 4
cap st "k_filter|k_light_ell|k_core_mark|k_label" 4
cap ct "k_relabel|k_hook|k_merge|k_jump" 6
ncu -i /tmp/prof_st_${TAG}.ncu-rep --page source --csv -k regex:k_filter > gpurun_out/source_filter_${TAG}.csv 2>/dev/null
ncu -i /tmp/prof_lr_${TAG}.ncu-rep --page source --csv > gpurun_out/source_lr_${TAG}.csv 2>/dev/null
ls -la gpurun_out/ | head -40
du -sh gpurun_out

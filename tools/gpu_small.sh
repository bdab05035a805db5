# small configs with/without the filter split; k_light_round DRAM bytes over all launches of a C4 step
mkdir -p gpurun_out
ARGS="--steps 10 --warmup 3 --no-e2e --no-cpu-baseline"
: > gpurun_out/small.jsonl
for c in C1 C2 C3; do
  timeout 300 python bench.py --config $c $ARGS 2>/dev/null | tail -1 >> gpurun_out/small.jsonl
  KDB_FILTER=0 timeout 300 python bench.py --config $c $ARGS 2>/dev/null | tail -1 >> gpurun_out/small.jsonl
done
echo "small rc=$?"
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_sector_hit_rate.pct --clock-control none \
  -k regex:"k_light_round" --csv --log-file gpurun_out/lr_dram.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/lr_dram.log 2>&1; echo "ncu rc=$?"

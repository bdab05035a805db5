# DRAM bytes of every kernel of one C4 step (ncu, 3 metrics): the per-step DRAM budget
mkdir -p gpurun_out
timeout 1200 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/dram_all.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/dram_all.log 2>&1
echo "ncu rc=$?"

set -x
free -g; nproc; lscpu | head -20; df -h /tmp /root | tail -3
nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv
KDB_TRACE=1 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/trace_c4.log 2> gpurun_out/trace_c4.err
echo rc=$?
tail -c 3000 gpurun_out/trace_c4.log
head -60 gpurun_out/trace_c4.err

# probe of the early light-round access pattern + a C4 trace (per-round counts)
mkdir -p gpurun_out
./tools/probe_round > gpurun_out/probe_round.log 2>&1; echo "probe rc=$?"
KDB_TRACE=1 timeout 600 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/trace_c4.log 2>&1; echo "trace rc=$?"

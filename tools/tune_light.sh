# per-round trace of one C4 step and a sweep of the light threshold column (KDB_LIGHT)
KDB_TRACE=1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/trace.json 2> gpurun_out/trace.err
for L in 6 8 12 14; do
  KDB_LIGHT=$L python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_L$L.json 2> gpurun_out/b_L$L.err
done

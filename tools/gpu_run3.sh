for cfg in "KDB_LIGHT=16 KDB_LAZY=0 KDB_FS=1" "KDB_LIGHT=16 KDB_LAZY=1 KDB_FS=1" "KDB_LIGHT=10 KDB_LAZY=0 KDB_FS=1"; do
env $cfg KDB_TRACE=1 timeout 900 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_x.log 2>&1; echo "== $cfg rc=$?"
grep "\[kdb\]" gpurun_out/bench_x.log | tail -$(grep -c "\[kdb\]" gpurun_out/bench_x.log | awk '{print int($1/2)}')
tail -1 gpurun_out/bench_x.log | python tools/show_bench.py
done

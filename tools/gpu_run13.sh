for b in 6 8 5; do
touch paper_2009_04552_b200/csrc/kdb.cu; make KDB_NVFLAGS=-DKDB_LR_MINB=$b paper_2009_04552_b200/lib/libkdb.so > /dev/null 2>&1
timeout 900 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline > gpurun_out/bench_b$b.log 2>&1; echo "bench minb=$b rc=$?"
tail -1 gpurun_out/bench_b$b.log | python tools/show_bench.py | head -2
done

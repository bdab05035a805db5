# light-round variant sweep (KDB_LRV), C4 bench lines
mkdir -p gpurun_out
for v in 0 1 2 3 4; do
  KDB_LRV=$v timeout 300 python bench.py --steps 5 --warmup 2 --no-e2e --no-cpu-baseline --out gpurun_out/lrv_$v.jsonl > gpurun_out/lrv_$v.log 2>&1; echo "lrv $v rc=$?"
done

# C4 single GPU + sim communicator at P = 2, 4, 8 (local-first stats for the scaling model)
mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --out gpurun_out/sim_1.jsonl > gpurun_out/sim_1.log 2>&1; echo "P1 rc=$?"
for P in 2 4 8; do
  timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --sim $P --out gpurun_out/sim_$P.jsonl > gpurun_out/sim_$P.log 2>&1; echo "sim $P rc=$?"
  KDB_LOCAL=0 timeout 600 python bench.py --steps 3 --warmup 2 --no-e2e --no-cpu-baseline --sim $P --out gpurun_out/simnolf_$P.jsonl > gpurun_out/simnolf_$P.log 2>&1; echo "sim nolf $P rc=$?"
done

# inertial order: per-round trace, launch list, sim-rank scaling lines
mkdir -p gpurun_out
TAG=${1:-ip}
KDB_TRACE=1 timeout 900 python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 1 > gpurun_out/${TAG}_trace.log 2>&1; echo "trace rc=$?"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --order inertial --no-cpu-baseline --no-e2e --steps 1 --warmup 0 > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu rc=$?"
for P in 4 8; do
timeout 900 python bench.py --order inertial --sim $P --no-cpu-baseline --no-e2e --steps 3 --out gpurun_out/${TAG}_sim.jsonl > gpurun_out/${TAG}_sim$P.log 2>&1; echo "sim $P rc=$?"
done

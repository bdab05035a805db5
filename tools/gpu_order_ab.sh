# A/B of the point order (generation vs inertial partition) on the bench path
mkdir -p gpurun_out
TAG=${1:-ord}
CFGS=${CFGS:-C4}
for c in $CFGS; do for o in ${ORDERS:-generation inertial}; do
timeout 900 python bench.py --config $c --order $o --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_${c}_${o}.log 2>&1; echo "$c $o rc=$?"
done; done

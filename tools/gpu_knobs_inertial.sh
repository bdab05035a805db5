# knob sweep on the default (inertial) C4 path: light column, gather width, L1 gathers, pipelining
mkdir -p gpurun_out
TAG=${1:-kn}
for v in "KDB_LIGHT=10" "KDB_LIGHT=8" "KDB_LIGHT=9" "KDB_LIGHT=11" "KDB_LIGHT=12" "KDB_GW=2" "KDB_L1GAT=1" "KDB_PIPE=1" "KDB_L2HINT=0" "KDB_LIGHT=10"; do
env $v timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_${TAG}.jsonl > gpurun_out/bench_${TAG}_$v.log 2>&1; echo "$v rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_$v.log | head -1)"
done

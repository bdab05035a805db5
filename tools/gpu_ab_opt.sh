# A/B of one tuning option on C4 (same box, alternating): bash tools/gpu_ab_opt.sh NAME VALUE_A VALUE_B [TAG]
mkdir -p gpurun_out
NAME=$1; A=$2; B=$3; TAG=${4:-ab}
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/${TAG}_parity.log 2>&1; echo "parity rc=$?"; tail -n 1 gpurun_out/${TAG}_parity.log
for rep in 1 2; do for v in $A $B; do
  env $NAME=$v timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/${TAG}.jsonl > gpurun_out/${TAG}_$v.log 2>&1
  echo "$NAME=$v rc=$? $(python -c "import json,sys; d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')][-1]; print('ms %.3f' % d['ms_per_step'], {k[:24]: round(v['ms_per_step'], 3) for k, v in list(d['kernels'].items())[:3]})" gpurun_out/${TAG}_$v.log)"
done; done

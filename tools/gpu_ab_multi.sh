# several option A/Bs on C4 in one call: bash tools/gpu_ab_multi.sh TAG "NAME=V ..." "NAME=V ..." ...
mkdir -p gpurun_out
TAG=$1; shift
for rep in 1 2; do i=0; for cfg in "$@"; do i=$((i+1))
  env $cfg timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/${TAG}.jsonl > gpurun_out/${TAG}_$i.log 2>&1
  echo "[$cfg] rc=$? $(python -c "import json,sys; d=[json.loads(l) for l in open(sys.argv[1]) if l.startswith('{')][-1]; print('ms %.3f' % d['ms_per_step'], {k[:24]: round(v['ms_per_step'], 3) for k, v in list(d['kernels'].items())[:2]})" gpurun_out/${TAG}_$i.log)"
done; done

# One gpurun call: per-config bench lines, the NCCL one-rank host path, the paper's edge set.
TAG=${1:-r01}
mkdir -p gpurun_out
ARGS="--steps 5 --warmup 3 --no-e2e --no-cpu-baseline"
: > gpurun_out/configs_${TAG}.jsonl
for c in C4 C3 C2 C1; do python bench.py --config $c $ARGS 2>/dev/null | tail -1 >> gpurun_out/configs_${TAG}.jsonl; done
python bench.py --config C4 --edge-cols 50 $ARGS 2>/dev/null | tail -1 > gpurun_out/ecM_${TAG}.jsonl
python bench.py --nccl1 $ARGS 2>/dev/null | tail -1 > gpurun_out/nccl1_${TAG}.jsonl
echo "configs rc=$?"

# the driver's other invocations with the final code: the reference arm, the 1-rank NCCL path, sim ranks, knng stage
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/arm_ref.log 2>&1; echo "reference rc=$?"; tail -c 600 gpurun_out/arm_ref.log
timeout 900 python bench.py --nccl1 --no-cpu-baseline --no-e2e --steps 3 > gpurun_out/arm_nccl1.log 2>&1; echo "nccl1 rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/arm_nccl1.log | head -1)"
timeout 900 python bench.py --stage knng > gpurun_out/arm_knng.log 2>&1; echo "knng rc=$?"; tail -c 400 gpurun_out/arm_knng.log

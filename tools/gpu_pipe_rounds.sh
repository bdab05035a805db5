# pipelined ELL chunk loads in selected light rounds only (rounds 3-4 scan ~6 entries per visit)
mkdir -p gpurun_out
for v in "KDB_PIPE_R0=0" "KDB_PIPE_R0=3 KDB_PIPE_R1=4" "KDB_PIPE_R0=3 KDB_PIPE_R1=5" "KDB_PIPE_R0=2 KDB_PIPE_R1=4" "KDB_PIPE_R0=4 KDB_PIPE_R1=6" "KDB_PIPE_R0=0"; do
env $v timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 20 > gpurun_out/pr.log 2>&1; echo "$v rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/pr.log | head -1) $(grep -o '"(k_light_round<4, [a-z]*, true>)": {"ms_per_step": [0-9.]*' gpurun_out/pr.log | tr '\n' ' ')"
done

# end-of-round measurements with the final code: bench line (C4, full), per-config lines, eps sweep,
# edge_cols = M, C5/4, then the profile (launch list with DRAM, ncu of the top kernels)
mkdir -p gpurun_out
timeout 900 python bench.py --out gpurun_out/final_bench.jsonl > gpurun_out/final_bench.log 2>&1; echo "bench rc=$?"
for c in C1 C2 C3; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/final_configs.jsonl > gpurun_out/final_$c.log 2>&1; echo "$c rc=$?"; done
timeout 900 python bench.py --config C5 --scale 0.25 --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/final_configs.jsonl > gpurun_out/final_C5q.log 2>&1; echo "C5q rc=$?"
timeout 900 python bench.py --eps-factors 1.0,1.25,1.5,2.0 --no-cpu-baseline --no-e2e --steps 5 --out gpurun_out/final_eps_sweep.jsonl > gpurun_out/final_eps.log 2>&1; echo "eps sweep rc=$?"
timeout 900 python bench.py --edge-cols M --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/final_edgecols.jsonl > gpurun_out/final_ec.log 2>&1; echo "edge_cols rc=$?"
bash tools/gpu_profile_r02c.sh r02f

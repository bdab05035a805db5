# session 5, last call: the final build on the generation order, and the reference arm's line
mkdir -p gpurun_out
timeout 600 python bench.py --order generation --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/bench_c4_generation_s5.jsonl > gpurun_out/bench_gen_s5.log 2>&1; echo "generation rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_gen_s5.log | head -1)"
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_reference_s5.log 2>&1; echo "reference rc=$?"; tail -n 1 gpurun_out/bench_reference_s5.log | cut -c1-400

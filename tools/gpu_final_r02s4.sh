# round 2, session 4: final measurements on the final code -- GPU suite, smoke, the bench line (C4, all
# defaults, e2e + cpu_baseline), per-config lines, eps sweep, edge_cols = M, launch list with DRAM of one
# step, ncu --set full of the first four light rounds (raw page + SASS source page)
mkdir -p gpurun_out
TAG=${1:-s4}
timeout 3000 python -m pytest tests -m gpu -q -x > gpurun_out/gputest_${TAG}.log 2>&1; echo "gpu tests rc=$?"; tail -n 2 gpurun_out/gputest_${TAG}.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke_${TAG}.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --out gpurun_out/bench_c4_${TAG}.jsonl > gpurun_out/bench_c4_${TAG}.log 2>&1; echo "bench rc=$?"
for c in C1 C2 C3; do timeout 900 python bench.py --config $c --no-cpu-baseline --no-e2e --steps 20 --out gpurun_out/configs_${TAG}.jsonl > gpurun_out/cfg_${c}_${TAG}.log 2>&1; echo "$c rc=$?"; done
timeout 900 python bench.py --config C5 --scale 0.25 --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/configs_${TAG}.jsonl > gpurun_out/cfg_C5q_${TAG}.log 2>&1; echo "C5q rc=$?"
timeout 900 python bench.py --eps-factors 1.0,1.25,1.5,2.0 --no-cpu-baseline --no-e2e --steps 5 --out gpurun_out/configs_${TAG}.jsonl > gpurun_out/cfg_eps_${TAG}.log 2>&1; echo "eps sweep rc=$?"
timeout 900 python bench.py --edge-cols M --no-cpu-baseline --no-e2e --steps 10 --out gpurun_out/configs_${TAG}.jsonl > gpurun_out/cfg_ec_${TAG}.log 2>&1; echo "edge_cols rc=$?"
ARGS="--steps 1 --warmup 0 --no-e2e --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    -k regex:"k_|cub|Radix|Scan|Select" --log-file gpurun_out/launches_${TAG}.csv python bench.py $ARGS > gpurun_out/ncu_launches_${TAG}.log 2>&1; echo "ncu launches rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_light_round" -s 0 -c 4 \
    -o /tmp/prof_lr_${TAG} python bench.py $ARGS > gpurun_out/ncu_lr_${TAG}.log 2>&1; echo "ncu lr rc=$?"
ncu -i /tmp/prof_lr_${TAG}.ncu-rep --page raw --csv > gpurun_out/raw_lr_${TAG}.csv 2>/dev/null
ncu -i /tmp/prof_lr_${TAG}.ncu-rep --page source --csv --print-source sass -k regex:k_light_round -s 1 -c 1 > gpurun_out/source_lr_${TAG}.csv 2>/dev/null
du -sh gpurun_out

# after the two-level global phase + filter policy: local-first tests, parity, configs, sim scaling
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_local_first.py tests/test_gpu_parity.py tests/test_eps_properties.py -x -q > gpurun_out/lf2_tests.log 2>&1; echo "tests rc=$?"
ARGS="--steps 5 --warmup 2 --no-e2e --no-cpu-baseline"
: > gpurun_out/cfg2.jsonl
for c in C1 C2 C3; do timeout 300 python bench.py --config $c $ARGS 2>/dev/null | tail -1 >> gpurun_out/cfg2.jsonl; done
timeout 300 python bench.py $ARGS --out gpurun_out/sim2_1.jsonl > /dev/null 2>&1
for P in 2 4 8; do timeout 600 python bench.py $ARGS --sim $P --out gpurun_out/sim2_$P.jsonl > gpurun_out/sim2_$P.log 2>&1; echo "sim $P rc=$?"; done

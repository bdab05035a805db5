# packed round 1 over a reused ELL (eps sweep): parity, sweep timing; partition determinism probe
mkdir -p gpurun_out
TAG=${1:-rp}
timeout 1500 python -m pytest tests/test_gpu_eps_reuse.py tests/test_gpu_parity.py tests/test_eps_properties.py tests/test_gpu_edge_cols.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
timeout 900 python bench.py --eps-factors 1.0,1.25,1.5,2.0 --no-cpu-baseline --no-e2e --steps 5 --out gpurun_out/bench_${TAG}_sweep.jsonl > gpurun_out/bench_${TAG}_sweep.log 2>&1; echo "sweep rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_sweep.log | head -1)"
timeout 900 python bench.py --no-cpu-baseline --no-e2e --steps 10 > gpurun_out/bench_${TAG}_c4.log 2>&1; echo "c4 rc=$? $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_${TAG}_c4.log | head -1)"
timeout 600 python tools/probe_partition_det.py C4 > gpurun_out/${TAG}_det.log 2>&1; echo "det rc=$?"; cat gpurun_out/${TAG}_det.log

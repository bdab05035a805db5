# two-level global-phase ids: local-first parity, then sim P=4/8 lines with and without
mkdir -p gpurun_out
TAG=${1:-gm}
timeout 1500 python -m pytest tests/test_gpu_local_first.py tests/test_gpu_parity.py -m gpu -x -q > gpurun_out/parity_${TAG}.log 2>&1; echo "parity rc=$?"; tail -n 2 gpurun_out/parity_${TAG}.log
for g in 1 0; do for P in 4 8; do KDB_GMAP=$g timeout 900 python bench.py --sim $P --no-cpu-baseline --no-e2e --steps 3 --out gpurun_out/${TAG}_sim_g$g.jsonl > gpurun_out/${TAG}_sim${P}_g$g.log 2>&1; echo "gmap=$g sim $P rc=$?"; done; done

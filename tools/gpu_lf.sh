# local-first contraction: dedicated tests + the sim / NCCL tests of the parity suite + smoke
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_local_first.py -x -q > gpurun_out/lf_tests.log 2>&1; echo "lf rc=$?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/lf_parity.log 2>&1; echo "parity rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/lf_smoke.log 2>&1; echo "smoke rc=$?"

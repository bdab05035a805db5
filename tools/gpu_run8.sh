timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q --durations=0 > gpurun_out/pytest_configs.log 2>&1; echo "pytest configs rc=$?"; tail -30 gpurun_out/pytest_configs.log

timeout 900 python -m pytest tests/test_gpu_knng.py -x -q > gpurun_out/pytest_knng.log 2>&1; echo "pytest knng rc=$?"; tail -3 gpurun_out/pytest_knng.log
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q --durations=0 -k "large" > gpurun_out/pytest_configs.log 2>&1; echo "pytest configs rc=$?"; tail -15 gpurun_out/pytest_configs.log

export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_exact.py -x -q -m gpu > gpurun_out/pytest_exact.log 2>&1; echo exact rc=$?; tail -25 gpurun_out/pytest_exact.log
timeout 900 python -u -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log

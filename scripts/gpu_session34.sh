timeout 1500 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log

export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 1200 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo all rc=$?; tail -5 gpurun_out/pytest_gpu_all.log
timeout 300 python -u -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/smoke.log

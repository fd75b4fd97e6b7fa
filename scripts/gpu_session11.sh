export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1 NCCL_DEBUG=WARN
timeout 400 python -u -m pytest tests/test_gpu_nccl_shards.py -x -q -rs > gpurun_out/pytest_nccl.log 2>&1; echo nccl rc=$?; tail -15 gpurun_out/pytest_nccl.log
timeout 300 python -u -m pytest tests -m gpu -x -q -k "facade" > gpurun_out/pytest_facade.log 2>&1; echo facade rc=$?; tail -3 gpurun_out/pytest_facade.log

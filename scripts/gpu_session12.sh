export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
timeout 600 python -u -m pytest tests/test_gpu_nccl_shards.py -x -q -rs > gpurun_out/pytest_p2p.log 2>&1; echo p2p rc=$?; tail -12 gpurun_out/pytest_p2p.log
timeout 900 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo all rc=$?; tail -4 gpurun_out/pytest_gpu.log

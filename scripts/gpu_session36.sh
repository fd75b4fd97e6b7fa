export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_gpu_nccl_shards.py tests/test_exact.py -q -m gpu -k "widened or argument" 2>&1 | tail -3
timeout 1500 python -u scripts/hilbert_c3.py c3 2>&1 | grep -v generated > gpurun_out/hilbert_c3.json; head -8 gpurun_out/hilbert_c3.json

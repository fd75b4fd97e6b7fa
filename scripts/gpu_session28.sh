export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_gpu_async_upload.py -x -q -m gpu 2>&1 | tail -15
timeout 600 python -u scripts/e2e_breakdown.py 2>&1 | grep -v generated

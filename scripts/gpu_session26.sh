export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 600 python -u scripts/e2e_breakdown.py 2>&1 | grep -v generated
timeout 600 nsys --version 2>/dev/null | head -1
timeout 900 python -u -m pytest tests/test_local_metrics.py tests/test_exact.py -q -m gpu -k "hilbert" 2>&1 | tail -2

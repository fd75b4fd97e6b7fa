timeout 900 python -u -m pytest tests/test_hll_statistics.py -q -m gpu 2>&1 | tail -3

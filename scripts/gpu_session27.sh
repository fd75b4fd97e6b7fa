timeout 900 python -u -m pytest tests/test_exact.py -q -m gpu -k contract 2>&1 | tail -15

timeout 1500 python -u scripts/hilbert_c3.py c3 2>&1 | grep -v generated

timeout 600 python -u scripts/step_overhead.py 2>&1 | grep -v generated

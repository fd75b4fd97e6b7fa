export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
( time ./tools/sb_hyperball analyze 486 486 0 1 1 20261017 7569 10 0 hyperball /tmp/c3.csv --interval ) 2>&1 | tail -5; ls -la /tmp/c3.csv; head -3 /tmp/c3.csv
( time ./tools/sb_hyperball analyze 212 212 60 3 10 20261017 1936 10 0 exact /tmp/c2.csv --interval ) 2>&1 | tail -5; head -2 /tmp/c2.csv
timeout 1500 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log

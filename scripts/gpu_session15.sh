export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 600 python -u -m pytest tests/test_local_metrics.py -x -q -m gpu > gpurun_out/pytest_local.log 2>&1; echo local rc=$?; tail -15 gpurun_out/pytest_local.log
timeout 300 python -u scripts/local_metrics_bench.py c2 > gpurun_out/local_c2.json 2> gpurun_out/local_c2.log; echo c2 rc=$?; cat gpurun_out/local_c2.json; tail -2 gpurun_out/local_c2.log
timeout 300 python -u scripts/local_metrics_bench.py c3 2000 > gpurun_out/local_c3s.json 2> gpurun_out/local_c3s.log; echo c3s rc=$?; cat gpurun_out/local_c3s.json; tail -2 gpurun_out/local_c3s.log

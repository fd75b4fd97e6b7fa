export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_local_metrics.py tests/test_graph_build.py tests/test_exact.py -x -q -m gpu > gpurun_out/pytest_local2.log 2>&1; echo tests rc=$?; tail -3 gpurun_out/pytest_local2.log
timeout 300 python -u scripts/local_metrics_bench.py c2 > gpurun_out/local_c2.json 2>/dev/null; echo c2 rc=$?; cat gpurun_out/local_c2.json
timeout 600 python -u scripts/local_metrics_bench.py c3 > gpurun_out/local_c3.json 2>/dev/null; echo c3 rc=$?; cat gpurun_out/local_c3.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_local2.csv python -u scripts/profile_local.py 117000 4096 > /dev/null 2>&1; echo launches rc=$?

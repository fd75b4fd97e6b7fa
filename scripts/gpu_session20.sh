export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_graph_build.py -x -q -m gpu > gpurun_out/pytest_build.log 2>&1; echo build rc=$?; tail -3 gpurun_out/pytest_build.log
timeout 900 python -u bench.py --local > gpurun_out/bench_r20.json 2> gpurun_out/bench_r20.log; echo bench rc=$?; grep "pipeline\|union avg\|Error\|error" gpurun_out/bench_r20.log | head

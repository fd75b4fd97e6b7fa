export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_graph_build.py -x -q -m gpu 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pipeline.csv python -u scripts/pipeline_profile.py c3 > gpurun_out/pipe.log 2>&1; echo rc=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pipeline_c2.csv python -u scripts/pipeline_profile.py c2 > gpurun_out/pipe2.log 2>&1; echo rc=$?

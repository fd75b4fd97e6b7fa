export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pipeline.csv python -u scripts/pipeline_profile.py c3 > gpurun_out/pipe.log 2>&1; echo rc=$?; tail -1 gpurun_out/pipe.log

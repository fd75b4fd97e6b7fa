export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_graph_build.py -x -q -m gpu 2>&1 | tail -2
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_pipeline.csv python -u scripts/pipeline_profile.py c3 > gpurun_out/pipe.log 2>&1; echo rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vis_rows -s 0 -c 2 -o gpurun_out/prof_vis_v3 python -u scripts/pipeline_profile.py c3 > gpurun_out/ncu_vis.log 2>&1; echo ncu2 rc=$?

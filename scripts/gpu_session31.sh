export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:union_interval -s 3 -c 1 -o gpurun_out/prof_interval_r31 python -u scripts/pipeline_profile.py c3 > gpurun_out/ncu_int.log 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vis_rows -s 0 -c 1 -o gpurun_out/prof_vis_r31 python -u scripts/pipeline_profile.py c3 > gpurun_out/ncu_vis.log 2>&1; echo ncu2 rc=$?

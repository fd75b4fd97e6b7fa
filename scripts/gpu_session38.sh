export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 1 -c 1 -o gpurun_out/prof_local_v2 python -u scripts/profile_local.py 117000 4096 > gpurun_out/ncu_local.log 2>&1; echo ncu rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:vis_rows -s 0 -c 2 -o gpurun_out/prof_vis_v2 python -u scripts/pipeline_profile.py c3 > gpurun_out/ncu_vis.log 2>&1; echo ncu2 rc=$?

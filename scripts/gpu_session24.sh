export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 300 python -u scripts/profile_local.py 117000 8192 > gpurun_out/local_prof_plain.log 2>&1; echo plain rc=$?; tail -1 gpurun_out/local_prof_plain.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:local_kernel -s 1 -c 1 -o gpurun_out/prof_local python -u scripts/profile_local.py 117000 4096 > gpurun_out/ncu_local.log 2>&1; echo ncu rc=$?; tail -2 gpurun_out/ncu_local.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_local.csv python -u scripts/profile_local.py 117000 4096 > /dev/null 2>&1; echo launches rc=$?

export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 900 python -u bench.py --local > gpurun_out/bench_r19.json 2> gpurun_out/bench_r19.log; echo bench rc=$?; grep "pipeline\|union avg" gpurun_out/bench_r19.log
SB_UNION_VARIANT=9 timeout 300 python -u bench.py --no-cpu --no-e2e --no-variants --no-pipeline --steps 2 --warmup 1 > gpurun_out/ab_v9.json 2> gpurun_out/ab_v9.log; echo v9 rc=$?; grep "union avg" gpurun_out/ab_v9.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:union_kernel -s 3 -c 1 -o gpurun_out/prof_union_kway python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline > gpurun_out/ncu_union.log 2>&1; echo ncu rc=$?; tail -3 gpurun_out/ncu_union.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python -u bench.py --profile --no-cpu --no-e2e --no-variants --no-pipeline > gpurun_out/ncu_launch.log 2>&1; echo launches rc=$?

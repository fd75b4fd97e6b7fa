export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
timeout 600 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc; tail -3 gpurun_out/pytest_gpu.log; [ $rc = 0 ] || exit 1
for v in 0 2 3 4; do
SB_UNION_VARIANT=$v timeout 300 python -u bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-variants > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.log; echo variant $v rc=$?; grep -E "runs x" gpurun_out/bench_v$v.log
done
timeout 900 python -u bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.log; echo bench full rc=$?; tail -14 gpurun_out/bench_full.log; cat gpurun_out/bench_full.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python -u bench.py --profile > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:union_kernel -s 2 -c 1 -o gpurun_out/prof_union_c3_v0 python -u bench.py --profile > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?

# fail-fast GPU session: correctness first, then bench, then profiles
export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python -u -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke rc=$rc; tail -5 gpurun_out/smoke.log; [ $rc = 0 ] || exit 1
timeout 900 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc; tail -25 gpurun_out/pytest_gpu.log
timeout 200 python -u bench.py --config c1 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.log; echo benchc1 rc=$?; tail -12 gpurun_out/bench_c1.log
timeout 600 python -u bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; echo benchc3 rc=$?; tail -25 gpurun_out/bench_c3.log; cat gpurun_out/bench_c3.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c3.csv python -u bench.py --profile > gpurun_out/ncu_launch.log 2>&1; echo ncu-launch rc=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:union_kernel -s 2 -c 1 -o gpurun_out/prof_union_c3 python -u bench.py --profile > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?; tail -3 gpurun_out/ncu_full.log

export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
timeout 120 python -u -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; rc=$?; echo smoke rc=$rc; tail -3 gpurun_out/smoke.log; [ $rc = 0 ] || exit 1
timeout 600 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc; tail -5 gpurun_out/pytest_gpu.log; [ $rc = 0 ] || exit 1
for s in warp tile; do
SB_UNION_SCHEDULE=$s timeout 300 python -u bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-variants > gpurun_out/bench_c3_$s.json 2> gpurun_out/bench_c3_$s.log; echo bench $s rc=$?; grep -E "runs x|t=1 |t=9 " gpurun_out/bench_c3_$s.log
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:union_kernel -s 2 -c 1 -o gpurun_out/prof_union_c3_tile python -u bench.py --profile > gpurun_out/ncu_full.log 2>&1; echo ncu-full rc=$?

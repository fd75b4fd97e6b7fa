export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
timeout 600 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc; tail -3 gpurun_out/pytest_gpu.log; [ $rc = 0 ] || exit 1
for v in 0 1 2 3 4; do
SB_UNION_VARIANT=$v timeout 300 python -u bench.py --steps 3 --warmup 2 --no-cpu --no-e2e --no-variants > gpurun_out/bench_v$v.json 2> gpurun_out/bench_v$v.log; echo variant $v rc=$?; grep -E "runs x" gpurun_out/bench_v$v.log
done
./tools/sb_hyperball synth 64 64 20 2 9 20261017 0 10 0 > gpurun_out/tool_c1.txt 2>&1; echo tool rc=$?; tail -4 gpurun_out/tool_c1.txt

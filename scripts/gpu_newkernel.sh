# Quick check of the union kernel on a B200: parity subset + C3 bench.
set -u
export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
mkdir -p gpurun_out
timeout 1200 python -u -m pytest tests/test_gpu_parity.py tests/test_gpu_async_upload.py -q -x > gpurun_out/pytest_parity.log 2>&1; echo "parity rc=$?"
tail -3 gpurun_out/pytest_parity.log
timeout 600 python -u bench.py --no-cpu --no-pipeline --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; echo "bench rc=$?"
grep "union=" gpurun_out/bench_c3.log | head -12
timeout 600 python -u -m pytest tests -q -m gpu -x --deselect tests/test_gpu_parity.py > gpurun_out/pytest_rest.log 2>&1; echo "rest rc=$?"
tail -3 gpurun_out/pytest_rest.log

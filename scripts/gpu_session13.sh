export SB_SYNC_TIMEOUT_S=120 PYTHONUNBUFFERED=1
nvidia-smi -L; nproc
timeout 1200 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?; tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -u -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?; tail -2 gpurun_out/smoke.log
timeout 900 python -u bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.log; echo bench rc=$?; cat gpurun_out/bench_default.json | head -c 600; echo
timeout 600 python -u bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.log; echo ref rc=$?; cat gpurun_out/bench_ref.json

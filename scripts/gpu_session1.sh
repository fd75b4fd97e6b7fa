set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 120 python -c "import __graft_entry__ as e; e.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -30 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c1 --steps 2 --warmup 1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.log; echo benchc1 rc=$?
tail -20 gpurun_out/bench_c1.log
timeout 900 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.log; echo benchc3 rc=$?
tail -30 gpurun_out/bench_c3.log; cat gpurun_out/bench_c3.json
nproc; lscpu | grep "Model name"

set -u
export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
mkdir -p gpurun_out
nproc > gpurun_out/nproc.txt; nvidia-smi -L >> gpurun_out/nproc.txt
timeout 1800 python -u -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2_w2_shared.json 2> gpurun_out/bench_c2_w2_shared.log; echo "w2 rc=$?"
timeout 600 python -u bench.py --config c2 --steps 3 --warmup 3 --no-cpu > gpurun_out/bench_c2_w1.json 2> gpurun_out/bench_c2_w1.log; echo "w1 rc=$?"

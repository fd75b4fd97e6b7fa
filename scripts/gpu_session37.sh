for i in 1 2 3; do timeout 900 python -u -m pytest tests/test_gpu_nccl_shards.py -q -m gpu -k "widened" -x 2>&1 | tail -30; done

timeout 1500 python -u scripts/shard_projection.py c3 2>&1 | grep -v generated > gpurun_out/shard_projection.json; cat gpurun_out/shard_projection.json

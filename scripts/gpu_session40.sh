timeout 1500 python -u scripts/accuracy_scale.py c2 c3 2>&1 | grep -v generated > gpurun_out/accuracy_scale.json; cat gpurun_out/accuracy_scale.json

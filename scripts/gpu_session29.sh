export SB_SYNC_TIMEOUT_S=600 PYTHONUNBUFFERED=1
timeout 1500 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo all rc=$?; tail -3 gpurun_out/pytest_gpu_all.log
timeout 900 python -u bench.py --local > gpurun_out/bench_r29.json 2> gpurun_out/bench_r29.log; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_r29.json')); print(d['value'], d['e2e'], d['pipeline']['interval']['total_s'], d['cpu_baseline']['value'])"

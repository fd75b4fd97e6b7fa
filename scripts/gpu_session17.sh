export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 900 python -u scripts/accuracy_table.py > gpurun_out/accuracy_table.json 2> gpurun_out/accuracy_table.log; echo acc rc=$?; python -c "
import json; d=json.load(open('gpurun_out/accuracy_table.json'))
for r in d['rows']: print(r)
print(d['means'])"
timeout 900 python -u -m pytest tests -q -m gpu > gpurun_out/pytest_gpu_all.log 2>&1; echo all rc=$?; tail -5 gpurun_out/pytest_gpu_all.log

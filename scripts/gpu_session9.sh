export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests -m gpu -x -q -k "interval or golden" > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc; tail -5 gpurun_out/pytest_gpu.log; [ $rc = 0 ] || exit 1
timeout 600 python -u bench.py --no-cpu --no-e2e > gpurun_out/bench_full.json 2> gpurun_out/bench_full.log; echo bench rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_full.json')); v=d['variants']
print('dense', d['ms_per_step'], 'skip', v['skip_unchanged']['seconds_per_run'], 'interval', v['interval']['seconds_per_run'], v['interval']['per_iteration_union_ms'], v['interval']['sum_d_identical_to_dense'])"
timeout 300 python -u bench.py --config c2 --no-cpu --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.log; echo bench c2 rc=$?; python -c "
import json; d=json.load(open('gpurun_out/bench_c2.json')); v=d['variants']
print('c2 dense ms/run', d['ms_per_step'], 'iters', d['config']['iterations'], 'skip', v['skip_unchanged']['seconds_per_run'], 'interval', v['interval']['seconds_per_run'], v['interval']['per_iteration_union_ms'])"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_interval.csv python -u -c "
import sys; sys.path.insert(0,'.')
from bench import build_graph
from paper_2604_08374_b200 import HyperBall
g=build_graph('c3'); h=HyperBall(g,10,None,interval=True); h.run()" > gpurun_out/ncu_il.log 2>&1; echo ncu-launch rc=$?
timeout 400 ncu --set full --clock-control none --import-source on -k regex:union_interval -s 2 -c 1 -o gpurun_out/prof_interval_c3c python -u -c "
import sys; sys.path.insert(0,'.')
from bench import build_graph
from paper_2604_08374_b200 import HyperBall
g=build_graph('c3'); h=HyperBall(g,10,None,interval=True); h.run()" > gpurun_out/ncu_interval.log 2>&1; echo ncu rc=$?

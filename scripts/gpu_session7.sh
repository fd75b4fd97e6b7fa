export SB_SYNC_TIMEOUT_S=90 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; rc=$?; echo pytest rc=$rc; tail -25 gpurun_out/pytest_gpu.log; [ $rc = 0 ] || exit 1
timeout 600 python -u bench.py --no-cpu > gpurun_out/bench_full.json 2> gpurun_out/bench_full.log; echo bench full rc=$?; tail -4 gpurun_out/bench_full.log; python -c "import json; d=json.load(open('gpurun_out/bench_full.json')); print(json.dumps(d['variants'], indent=1)); print(d['value'], d['e2e'])"
timeout 400 ncu --set full --clock-control none --import-source on -k regex:union_interval -s 2 -c 1 -o gpurun_out/prof_interval_c3 python -u -c "
import sys; sys.path.insert(0,'.')
from bench import build_graph
from paper_2604_08374_b200 import HyperBall
g=build_graph('c3'); h=HyperBall(g,10,None,interval=True); h.run(); print(h.stats())" > gpurun_out/ncu_interval.log 2>&1; echo ncu rc=$?

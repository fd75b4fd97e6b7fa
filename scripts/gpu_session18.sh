export SB_SYNC_TIMEOUT_S=300 PYTHONUNBUFFERED=1
timeout 900 python -u -m pytest tests/test_graph_build.py tests/test_exact.py -x -q -m gpu > gpurun_out/pytest_build.log 2>&1; echo build rc=$?; tail -25 gpurun_out/pytest_build.log
timeout 600 python -u -c "
import sys, time, hashlib; sys.path.insert(0,'.')
import numpy as np
from paper_2604_08374_b200 import DeviceGraph, grid_mask, HyperBall
from bench import build_graph
for cfg, (rows, cols, k, a, b, seed, r2) in (('c2', (212, 212, 60, 3, 10, 20261017, 44*44)), ('c3', (486, 486, 0, 1, 1, 20261017, 87*87))):
    m = grid_mask(rows, cols, k, a, b, seed)
    DeviceGraph.from_grid(grid_mask(16,16,0,1,1,1), 9)  # warm-up
    t0 = time.perf_counter(); dg = DeviceGraph.from_grid(m, r2); t1 = time.perf_counter()
    off, deg, st = dg.download()
    t2 = time.perf_counter(); ref = build_graph(cfg); t3 = time.perf_counter()
    same = np.array_equal(off, ref.offsets) and np.array_equal(deg, ref.degrees) and np.array_equal(st, ref.stream)
    print(cfg, 'gpu build %.3f s' % (t1 - t0), 'cpu build %.3f s' % (t3 - t2), 'identical', same, dg.n, dg.edges, flush=True)
" > gpurun_out/build_timing.log 2>&1; echo timing rc=$?; cat gpurun_out/build_timing.log | grep -v generated

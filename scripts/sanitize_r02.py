"""Small runs of the round-2 union paths for compute-sanitizer (memcheck /
racecheck / synccheck): the 16-node group path (forced `group` schedule) at
p = 9 / 10 / 12 incl. skip mode and a 2-window id span, the per-node D16 feeder
at p = 4 / 5 / 6 / 8 (paired p = 4 rows), the p >= 9 per-node items, the
asynchronous chunked upload feeding the group path, and the wavefront first
run in dense and interval mode.  Results are checked against
the plain schedule so a silent corruption also fails the run."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, HyperBall  # noqa: E402

g = CompressedCsr.synth_grid(72, 72, 12, 2, 5, 11, 20 * 20)     # ~1,200 neighbours per row, one id window
wide = CompressedCsr.synth_grid(40, 420, 20, 2, 6, 7, 14 * 14)   # id span > 8,192: several windows per group
for graph in (g, wide):
    dg = DeviceGraph(graph)
    for p in (4, 5, 6, 8, 9, 10, 12):
        ref = None
        for sched in ("items", "auto", "group"):
            for skip in ((False, True) if p in (6, 10) else (False,)):
                h = HyperBall(dg, p, 3, schedule=sched, skip_unchanged=skip)
                h.run()
                r = h.registers()
                if ref is None:
                    ref = r
                assert np.array_equal(r, ref), (p, sched, skip)
h = HyperBall(DeviceGraph(g, async_upload=True), 10, None, schedule="group")
h.run()
h.registers()
# the wavefront first run (dense and interval: run index per chunk, tables per pass and chunk)
w = CompressedCsr.synth_grid(150, 150, 30, 2, 6, 5, 6 * 6)
for interval in (False, True):
    ref = HyperBall(w, 10, None)
    ref.run()
    h = HyperBall(DeviceGraph(w, async_upload=True), 10, None, wavefront=True, interval=interval)
    h.run()
    assert np.array_equal(h.registers(), ref.registers()), interval
print("ok")

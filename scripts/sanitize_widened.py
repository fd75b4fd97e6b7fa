"""Small runs of the widened device passes for compute-sanitizer (memcheck /
racecheck / synccheck): local metrics (smem + global scratch), exact BFS
(dense + interval, 2 source blocks), on-device grid build."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, ExactBfs, grid_mask  # noqa: E402

g = CompressedCsr.synth_grid(70, 70, 20, 2, 6, 5, 8 * 8)
dg = DeviceGraph(g)
dg.local_metrics()
for interval in (False, True):
    x = ExactBfs(dg, None, interval=interval)
    x.run()
    x.result()
b = DeviceGraph.from_grid(grid_mask(40, 60, 25, 1, 6, 3), 10 * 10)
b.local_metrics()
b.grid_info()
print("ok")

"""Small runs of the device passes for compute-sanitizer (memcheck / racecheck /
synccheck): local metrics (smem + global scratch), exact BFS (dense + interval,
2 source blocks), on-device grid build, the asynchronous chunked upload with
the pipelined first pass, and the bit-serial dense union for p = 6 / 10 / 12."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, ExactBfs, HyperBall, grid_mask  # noqa: E402

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
for p in (6, 10, 12):
    h = HyperBall(DeviceGraph(g, async_upload=True), p, None)
    h.run()
    h.registers()
h = HyperBall(DeviceGraph(g, async_upload=True), 10, None, interval=True)
h.run()
# local metrics: both |N2| methods, shared / global scratch, the wide-window 1024-thread CTA
import os as _os  # noqa: E402
for n2 in ("bfs", "bitmap"):
    _os.environ["SB_LOCAL_N2"] = n2
    DeviceGraph(g).local_metrics()
    DeviceGraph.from_grid(grid_mask(24, 3000, 200, 2, 6, 5), 20 * 20).local_metrics(0, 512)
_os.environ.pop("SB_LOCAL_N2")
print("ok")

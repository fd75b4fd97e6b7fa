"""The on-device pipeline once (mask -> graph in HBM -> interval HyperBall -> metrics), for ncu launch lists."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import CONFIGS  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HyperBall, grid_mask  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
r, c, k, a, b, seed, rad2, _ = CONFIGS[cfg]
dg = DeviceGraph.from_grid(grid_mask(r, c, k, a, b, seed), rad2)
h = HyperBall(dg, 10, None, interval=True)
h.run()
m = h.metrics(dg.node_count_of_component(), dg.degrees())
print("ok", dg.n)

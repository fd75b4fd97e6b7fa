"""Dense union ms/pass per schedule on the city-scale raster (1650^2, radius 30,
12,000 buildings) and the Valdivia-sized one (1800^2, radius 80, 6,500
buildings): is the group path's density rule right at city scale?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2604_08374_b200 import DeviceGraph, HyperBall, grid_mask  # noqa: E402

for side, R, rects, depth in ((1650, 30, 12000, 4), (1800, 80, 6500, 3)):
    dg = DeviceGraph.from_grid(grid_mask(side, side, rects, 4, 16, 20261017), R * R)
    row = {"grid": side, "radius": R, "nodes": dg.n, "edges": dg.edges}
    for sched in ("auto", "group", "items"):
        hb = HyperBall(dg, 10, depth, schedule=sched)
        hb.run()
        hb.reset()
        hb.run()
        row[sched] = round(sum(s["union_ms"] for s in hb.stats()) / len(hb.stats()), 2)
        del hb
    print(json.dumps(row), flush=True)
    del dg

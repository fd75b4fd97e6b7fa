"""City-scale run (paper §5: 2.7 M-cell Valdivia analysis on one GPU):
usage: python scripts/city_scale.py SIDE RADIUS RECTS [DEPTH]
a SIDE x SIDE raster with RECTS building-like rectangular obstacles (4-16
cells), visibility radius RADIUS cells, built on the device
(sb_graph_build_grid), analysed with HyperBall (interval and dense) at p = 10
to DEPTH (0 = convergence), plus exact local metrics for every node.
Prints one JSON object with the timings."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2604_08374_b200 import DeviceGraph, HyperBall, grid_mask  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 1650
R = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rects = int(sys.argv[3]) if len(sys.argv) > 3 else 12000
depth = int(sys.argv[4]) if len(sys.argv) > 4 and int(sys.argv[4]) > 0 else None
mask = grid_mask(side, side, rects, 4, 16, 20261017)
DeviceGraph.from_grid(grid_mask(8, 8), 4)  # context + module load
t0 = time.perf_counter()
dg = DeviceGraph.from_grid(mask, R * R)
t_build = time.perf_counter() - t0
nv = dg.node_count_of_component()
out = {"grid": f"{side}x{side}", "blocked_cells": int(mask.sum()), "radius_cells": R, "depth_limit": depth,
       "nodes": dg.n,
       "edges": dg.edges, "stream_bytes": dg.stream_bytes_local, "components": int(len(np.unique(nv))),
       "build_s": t_build}
for mode in ("interval", "dense"):
    hb = HyperBall(dg, 10, depth, interval=(mode == "interval"))
    t0 = time.perf_counter()
    it = hb.run()
    t_run = time.perf_counter() - t0
    st = hb.stats()
    m = hb.metrics(nv, dg.degrees())
    out[mode] = dict(iterations=it, seconds=t_run, union_ms_mean=float(np.mean([s["union_ms"] for s in st])),
                     mean_md=float(np.nanmean(m["md"])),
                     edge_register_updates_per_s=it * dg.edges * 1024 / t_run)
    del hb
t0 = time.perf_counter()
lm = dg.local_metrics()
out["local_metrics_all_nodes_s"] = time.perf_counter() - t0
out["mean_clustering"] = float(np.nanmean(lm["clustering"]))
print(json.dumps(out, indent=1))

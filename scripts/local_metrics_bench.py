"""Times the exact local-metrics pass (sb_local_metrics) on a bench config.

usage: python scripts/local_metrics_bench.py [c1|c2|c3] [max_nodes]
Prints one JSON line: nodes, seconds (host wall around the synchronous C-ABI
call, run index already built), run count and per-node means."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
cap = int(sys.argv[2]) if len(sys.argv) > 2 else 0
g = build_graph(cfg)
dg = DeviceGraph(g)
n = g.n if not cap else min(cap, g.n)
dg.local_metrics(0, min(64, n))  # builds the run index
t0 = time.perf_counter()
m = dg.local_metrics(0, n)
dt = time.perf_counter() - t0
print(json.dumps({"config": cfg, "nodes": n, "graph_nodes": g.n, "edges": g.edges, "seconds": dt,
                  "nodes_per_s": n / dt, "mean_n2": float(np.mean(m["n2"])),
                  "mean_clustering": float(np.nanmean(m["clustering"])),
                  "mean_control": float(np.mean(m["control"]))}))

"""Times the exact bit-parallel BFS (sb_exact_*) on a bench config.

usage: python scripts/exact_bench.py c2|c3 [dense|interval] [log2_block]
Prints one JSON line: seconds (wall around the synchronous run, run index
built beforehand), union kernel time, launches, max depth, bytes/iteration."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, ExactBfs  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
mode = sys.argv[2] if len(sys.argv) > 2 else "interval"
lb = int(sys.argv[3]) if len(sys.argv) > 3 else 12
g = build_graph(cfg)
dg = DeviceGraph(g)
x = ExactBfs(dg, None, log2_block=lb, interval=(mode == "interval"))
x.run(0, min(64, g.n))  # warm-up (builds the run index in interval mode)
x = ExactBfs(dg, None, log2_block=lb, interval=(mode == "interval"))
t0 = time.perf_counter()
md = x.run()
dt = time.perf_counter() - t0
st = x.stats()
r = x.result(with_hist=False)
nv = g.node_count_of_component()
print(json.dumps({"config": cfg, "mode": mode, "log2_block": lb, "nodes": g.n, "edges": g.edges, "seconds": dt,
                  "union_ms_total": st["union_ms"], "union_launches": st["union_launches"], "max_depth": md,
                  "reach_is_component_size": bool(np.array_equal(r["reach"], nv)),
                  "mean_md_exact": float(np.mean(r["sum_d"] / np.maximum(nv - 1.0, 1.0))),
                  "source_bits_per_s": g.n * float(g.edges) / dt}))

"""Hilbert renumbering at C3 scale: reorder time, compressed size,
union ms/iteration raster vs Hilbert (dense + interval), and the permutation-
equivariance of the full-depth result (sum_d byte-identical after inverse permutation)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import HyperBall  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
g = build_graph(cfg)
t0 = time.perf_counter()
h = g.hilbert_reorder()
t_reorder = time.perf_counter() - t0
inv = h.hilbert_inverse.astype(np.int64)
out = {"config": cfg, "nodes": g.n, "edges": g.edges, "stream_raster": g.stream_len,
       "stream_hilbert": h.stream_len, "reorder_s_host": t_reorder}
for mode in ("dense", "interval"):
    res = {}
    for name, gg in (("raster", g), ("hilbert", h)):
        hb = HyperBall(gg, 10, None, interval=(mode == "interval"))
        hb.run()
        hb.reset()
        it = hb.run()
        st = hb.stats()
        res[name] = dict(iterations=it, union_ms=float(np.mean([s["union_ms"] for s in st])),
                         sum_d=hb.state().sum_d)
    out[mode] = {k: {kk: vv for kk, vv in v.items() if kk != "sum_d"} for k, v in res.items()}
    out[mode]["sum_d_equivariant"] = bool(np.array_equal(res["hilbert"]["sum_d"], res["raster"]["sum_d"][inv]))
print(json.dumps(out, indent=1))

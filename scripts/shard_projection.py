"""Multi-GPU projection from one GPU: C3 split into G edge-balanced node-range
shards (the partition bench.py --gpus G uses), each shard's union + estimate
timed on the device one after another (sb_hb_exchange_local between
iterations).  The slowest shard per iteration bounds the G-GPU iteration time
(+ the exchange, not measurable here).  PROJECTION, not a multi-GPU measurement."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HyperBall  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
g = build_graph(cfg)
out = {"config": cfg, "nodes": g.n, "edges": g.edges, "note": __doc__.split("\n")[0]}
ref_sum = None
for G in (1, 2, 4, 8):
    b = g.partition(G)
    shards = [HyperBall(DeviceGraph(g, node_range=(int(b[r]), int(b[r + 1]))), 10, None,
                        node_range=(int(b[r]), int(b[r + 1]))) for r in range(G)]
    while True:
        mx = max(h.step_compute() for h in shards)
        HyperBall.exchange_local(shards)
        fin = [h.step_finish(mx)[1] for h in shards]
        if fin[0]:
            break
    per = np.array([[s["union_ms"] + s["estimate_ms"] for s in h.stats()] for h in shards])  # G x iters
    sd = np.concatenate([h.state().sum_d for h in shards])
    if ref_sum is None:
        ref_sum = sd
    out[G] = dict(iterations=int(per.shape[1]), shard_edges=[int(x.graph.edges_local) for x in shards],
                  max_shard_ms_per_iter=float(per.max(0).mean()), mean_shard_ms_per_iter=float(per.mean()),
                  imbalance=float(per.max(0).mean() / per.mean()),
                  sum_d_identical_to_1_shard=bool(np.array_equal(sd, ref_sum)))
    del shards
base = out[1]["max_shard_ms_per_iter"]
for G in (2, 4, 8):
    out[G]["projected_speedup_compute_only"] = base / out[G]["max_shard_ms_per_iter"]
print(json.dumps(out, indent=1))

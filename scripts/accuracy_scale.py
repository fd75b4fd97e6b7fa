"""HyperBall vs the exact GPU BFS at bench scale (C2, C3): paper Table 1 at city size.
Prints one JSON object: per config and precision, MD Pearson r, median relative MD
error, IHH Spearman rho (validate.compare), plus exact/HyperBall run times."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, ExactBfs, HyperBall, metrics_from_sums, validate  # noqa: E402

out = {}
for cfg in sys.argv[1:] or ["c2", "c3"]:
    g = build_graph(cfg)
    dg = DeviceGraph(g)
    nv, deg = g.node_count_of_component(), g.degrees
    t0 = time.perf_counter()
    x = ExactBfs(dg, None, interval=True)
    x.run()
    ex = x.result(with_hist=False)
    t_exact = time.perf_counter() - t0
    exm = metrics_from_sums(ex["sum_d"], ex["sum_d2"], nv, deg)
    rows = {}
    for p in (8, 10, 12):
        t0 = time.perf_counter()
        hb = HyperBall(dg, p, None, interval=True)
        it = hb.run()
        m = hb.metrics(nv, deg)
        t_hb = time.perf_counter() - t0
        rep = {r["metric"]: r for r in validate.compare(m, exm)}
        rows[p] = dict(iterations=it, seconds=t_hb, md_pearson_r=rep["md"]["pearson_r"],
                       md_median_rel_err=rep["md"]["median_rel_err"], ihh_spearman=rep["ihh"]["spearman_rho"],
                       tekl_pearson_r=rep["tekl"]["pearson_r"])
    out[cfg] = dict(nodes=g.n, edges=g.edges, exact_seconds=t_exact, exact_mean_md=float(np.nanmean(exm["md"])),
                    hyperball=rows)
print(json.dumps(out, indent=1))

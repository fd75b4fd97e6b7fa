#!/usr/bin/env python
"""BASELINE configs C4 (precision sweep on C2) and C5 (depth sweep on C3) on
one GPU.  Writes one JSON document (stdout) with, per point: iterations,
device seconds per full run (median of 3), union ms per iteration, dense
edge-register updates/s and algorithmic GB/s, for the dense kernel and (p>=10)
the interval variant.  Not part of the driver's bench contract; evidence for
DESIGN.md / profiles/."""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from bench import alg_bytes_per_iter, build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HllParams, HyperBall  # noqa: E402


def time_runs(hb, reps=3):
    s = torch.cuda.ExternalStream(hb.stream_handle())
    hb.reset()
    it = hb.run()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        hb.reset()
        it = hb.run()
        e1.record(s)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    st = hb.stats()
    return it, statistics.median(ts), statistics.mean(x["union_ms"] for x in st)


def point(g, dg, p, depth, interval):
    hb = HyperBall(dg, HllParams(p), depth, interval=interval)
    it, sec, ums = time_runs(hb)
    m = 1 << p
    out = {"p": p, "depth": depth, "mode": "interval" if interval else "dense", "iterations": it,
           "seconds_per_run": sec, "union_ms_per_iter": ums,
           "edge_register_updates_per_s": it * g.edges * m / sec,
           "alg_gbs": alg_bytes_per_iter(g.n, g.edges, g.stream_len, p) * it / sec / 1e9}
    print(json.dumps(out), file=sys.stderr, flush=True)
    return out


def main():
    torch.cuda.set_device(0)
    res = {"c4": [], "c5": []}
    g2 = build_graph("c2")
    dg2 = DeviceGraph(g2, 0)
    res["c4_graph"] = {"nodes": g2.n, "edges": g2.edges, "stream_bytes": g2.stream_len}
    for p in (4, 6, 8, 10, 12, 14):
        res["c4"].append(point(g2, dg2, p, None, False))
        res["c4"].append(point(g2, dg2, p, None, True))
    del dg2
    g3 = build_graph("c3")
    dg3 = DeviceGraph(g3, 0)
    res["c5_graph"] = {"nodes": g3.n, "edges": g3.edges, "stream_bytes": g3.stream_len}
    for d in (3, 5, 10, None):
        res["c5"].append(point(g3, dg3, 10, d, False))
        res["c5"].append(point(g3, dg3, 10, d, True))
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

"""Phase breakdown of the end-to-end C-ABI path on small graphs (C1, C2): where the
fixed per-call cost goes when the HyperBall run itself is only milliseconds."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HllParams, HyperBall  # noqa: E402

for cfg, depth in (("c1", 3), ("c2", None)):
    g = build_graph(cfg)
    g.pin(True)
    P = HllParams(10)
    for rep in range(8):
        t0 = time.perf_counter()
        dg = DeviceGraph(g, 0, async_upload=True)
        t1 = time.perf_counter()
        h = HyperBall(dg, P, depth)
        t2 = time.perf_counter()
        it = h.run()
        t3 = time.perf_counter()
        s = h.state()
        t4 = time.perf_counter()
        del h
        t5 = time.perf_counter()
        del dg
        torch.cuda.synchronize()
        t6 = time.perf_counter()
        print(f"{cfg} rep {rep}: graph_create {1e3 * (t1 - t0):.2f} ms, hb_create {1e3 * (t2 - t1):.2f} ms, "
              f"run {1e3 * (t3 - t2):.2f} ms ({it} it), read_state {1e3 * (t4 - t3):.2f} ms, "
              f"hb_destroy {1e3 * (t5 - t4):.2f} ms, graph_destroy {1e3 * (t6 - t5):.2f} ms, "
              f"total {1e3 * (t6 - t0):.2f} ms", flush=True)

"""Phase breakdown of the end-to-end C-ABI path on C3 (host CSR -> HBM -> run -> read-back),
dense (sync / async upload) and interval (async upload: the run index is counted per upload chunk)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HllParams, HyperBall  # noqa: E402

g = build_graph("c3")
g.pin(True)
P = HllParams(10)
for rep in range(9):
    interval = rep >= 6
    t0 = time.perf_counter()
    dg = DeviceGraph(g, 0, async_upload=rep >= 3)
    t1 = time.perf_counter()
    h = HyperBall(dg, P, None, interval=interval)
    t2 = time.perf_counter()
    it = h.run()
    t3 = time.perf_counter()
    s = h.state()
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    mode = "interval async" if interval else ("dense async" if rep >= 3 else "dense sync")
    print(f"rep {rep} ({mode}): graph_create {t1 - t0:.3f} s, hb_create {t2 - t1:.3f} s, run {t3 - t2:.3f} s "
          f"({it} it), read_state {t4 - t3:.3f} s, total {t4 - t0:.3f} s", flush=True)
    del h, dg, s

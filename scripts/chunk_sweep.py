"""A-B sweep of the asynchronous upload's chunk count (SB_UPLOAD_CHUNKS) at C3:
end-to-end time of the wavefront first run (dense and interval), host CSR ->
HBM -> run -> read-back, and the final registers' hash against a synchronous run.
Needs an A-B build (`make -B NVEXTRA=-DSB_AB_UPLOAD_CHUNKS`): the product library
has no environment switch and always uses 16 chunks."""
import hashlib
import json
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
ref = {}
for interval in (False, True):
    h = HyperBall(DeviceGraph(g, 0), P, None, interval=interval)
    h.run()
    ref[interval] = hashlib.sha256(h.registers().tobytes()).hexdigest()
    del h
out = []
for k in [int(x) for x in (sys.argv[1:] or ["16", "24", "32", "48", "64"])]:
    os.environ["SB_UPLOAD_CHUNKS"] = str(k)
    for interval in (False, True):
        ts, same = [], True
        for rep in range(4):
            t0 = time.perf_counter()
            dg = DeviceGraph(g, 0, async_upload=True)
            h = HyperBall(dg, P, None, interval=interval)
            h.run()
            s = h.state()
            torch.cuda.synchronize()
            ts.append(time.perf_counter() - t0)
            same &= hashlib.sha256(h.registers().tobytes()).hexdigest() == ref[interval]
            del h, dg, s
        r = dict(chunks=k, mode="interval" if interval else "dense", e2e_s=[round(t, 4) for t in ts],
                 best_s=round(min(ts[1:]), 4), identical=same)
        print(json.dumps(r), flush=True)
        out.append(r)

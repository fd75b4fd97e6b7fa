"""Asynchronous upload + wavefront first run (dense or interval) on random small
grids, final state vs the oracle; for compute-sanitizer runs of the wavefront
on the graph shapes the randomised campaign draws.
usage: python scripts/wave_fuzz.py n_cases seed [big | rows cols rects rmin rmax radius2 gseed p depth]
("big": 60-160 rows/cols, radius^2 20-400, p 4-12 -- more chunks per row reach)"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (parity checker: test infrastructure)
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, ExactBfs, HyperBall  # noqa: E402

O = oracle.reference() if oracle.reference_available() else oracle.port()
n_cases, rng = int(sys.argv[1]), np.random.default_rng(int(sys.argv[2]))
big = sys.argv[3:] == ["big"]
fixed = [] if big else [int(x) if x != "None" else None for x in sys.argv[3:]]
bad = 0
for case in range(n_cases):
    if fixed:
        rows, cols, rects, rmin, rmax, radius2, gseed, p, depth = fixed
    elif big:
        rows, cols = int(rng.integers(60, 161)), int(rng.integers(60, 161))
        rects = int(rng.integers(0, rows * cols // 40 + 1))
        rmin = int(rng.integers(1, 4))
        rmax = rmin + int(rng.integers(0, 8))
        radius2 = int(rng.integers(20, 401))
        gseed = int(rng.integers(1, 2**31))
        p = int(rng.integers(4, 13))
        depth = None if rng.random() < 0.5 else int(rng.integers(1, 8))
    else:
        rows, cols = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        rects = int(rng.integers(0, rows * cols // 20 + 1))
        rmin = int(rng.integers(1, 4))
        rmax = rmin + int(rng.integers(0, 6))
        radius2 = 0 if rng.random() < 0.4 else int(rng.integers(1, 200))
        gseed = int(rng.integers(1, 2**31))
        p = int(rng.integers(4, 17)) if rng.random() < 0.5 else 10
        depth = None if rng.random() < 0.5 else int(rng.integers(1, 6))
    try:
        g = CompressedCsr.synth_grid(rows, cols, rects, rmin, rmax, gseed, radius2)
    except RuntimeError:
        continue
    ref = O.hb_run(g, p, depth_limit=depth)
    for interval in (True, False):
        h = HyperBall(DeviceGraph(g, async_upload=True), p, depth, wavefront=True, interval=interval)
        h.run()
        st = h.state()
        ok = st.t == ref["iterations"] and np.array_equal(h.registers(), ref["registers"])
        ok &= np.array_equal(st.sum_d, ref["sum_d"]) and np.array_equal(st.c_curr, ref["c"])
        if not ok:
            bad += 1
            print(json.dumps(dict(rows=rows, cols=cols, rects=rects, rmin=rmin, rmax=rmax, radius2=radius2,
                                  seed=gseed, p=p, depth=depth, interval=interval, n=g.n)), flush=True)
        del h
    if case % 3 == 0:  # the run index's other users over an asynchronous upload
        ra, rb = DeviceGraph(g, async_upload=True).local_metrics(), DeviceGraph(g).local_metrics()
        ok = all(np.array_equal(ra[k], rb[k], equal_nan=ra[k].dtype.kind == "f") for k in rb)
        xa, xb = ExactBfs(DeviceGraph(g, async_upload=True), depth, interval=True), ExactBfs(DeviceGraph(g), depth)
        xa.run()
        xb.run()
        ea, eb = xa.result(), xb.result()
        ok &= all(np.array_equal(ea[k], eb[k]) for k in ("sum_d", "sum_d2", "reach"))
        if not ok:
            bad += 1
            print(json.dumps(dict(rows=rows, cols=cols, rects=rects, rmin=rmin, rmax=rmax, radius2=radius2,
                                  seed=gseed, depth=depth, what="local/exact", n=g.n)), flush=True)
print(json.dumps(dict(cases=n_cases, mismatches=bad)))

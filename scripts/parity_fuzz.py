"""Randomised parity campaign: random grid graphs (size, obstacles, radius),
random p in [4, 16], random depth limit, random mode (dense / skip / interval /
sharded / asynchronous upload with the wavefront first run) and schedule (auto /
group / items), GPU vs the oracle after EVERY iteration (the wavefront run: its
final state and every max increase); plus exact local metrics and the exact BFS
on the same graph.  usage: python scripts/parity_fuzz.py [n_cases] [seed] [big]
("big": 100-160 rows/cols, radius^2 20-400, p 8-12 -- graphs over the auto
schedule's group-path threshold, so "auto" picks the 16-node group path)
Prints one JSON summary (cases, failures with their parameters)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (parity checker: test infrastructure)
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, HyperBall, exact_bfs_all  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 100
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 12345)
O = oracle.reference() if oracle.reference_available() else oracle.port()
P = oracle.port()
fails, done, t_start = [], 0, time.time()
big = len(sys.argv) > 3 and sys.argv[3] == "big"
for case in range(n_cases):
    if big:
        rows, cols = int(rng.integers(100, 161)), int(rng.integers(100, 161))
        rects = int(rng.integers(0, rows * cols // 40 + 1))
        rmin = int(rng.integers(1, 4))
        rmax = rmin + int(rng.integers(0, 8))
        radius2 = int(rng.integers(20, 401))
        seed = int(rng.integers(1, 2**31))
        p = int(rng.integers(8, 13))
    else:
        rows, cols = int(rng.integers(2, 60)), int(rng.integers(2, 60))
        rects = int(rng.integers(0, rows * cols // 20 + 1))
        rmin = int(rng.integers(1, 4))
        rmax = rmin + int(rng.integers(0, 6))
        radius2 = 0 if rng.random() < 0.4 else int(rng.integers(1, 200))
        seed = int(rng.integers(1, 2**31))
        p = int(rng.integers(4, 17)) if rng.random() < 0.5 else 10
    depth = None if rng.random() < 0.5 else int(rng.integers(1, 6))
    mode = rng.choice(["dense", "skip", "interval", "shards", "async"])
    sched = str(rng.choice(["auto", "group", "items"])) if mode in ("dense", "skip") else "auto"
    params = dict(rows=rows, cols=cols, rects=rects, rmin=rmin, rmax=rmax, radius2=radius2, seed=seed, p=p,
                  depth=depth, mode=str(mode), schedule=sched)
    try:
        g = CompressedCsr.synth_grid(rows, cols, rects, rmin, rmax, seed, radius2)
    except RuntimeError:
        continue  # every cell blocked
    try:
        n = g.n
        cur, c_prev = O.hb_init(n, p)
        nxt = np.zeros_like(cur)
        c_cur, sd, sd2 = np.zeros(n), np.zeros(n), np.zeros(n)
        if mode == "async":
            h = HyperBall(DeviceGraph(g, async_upload=True), p, depth, wavefront=True,
                          interval=bool(rng.random() < 0.5))
            h.run()
            ref = O.hb_run(g, p, depth_limit=depth)
            st = h.state()
            ok = st.t == ref["iterations"] and np.array_equal(h.registers(), ref["registers"])
            ok &= np.array_equal(st.sum_d, ref["sum_d"]) and np.array_equal(st.c_curr, ref["c"])
            if not ok:
                raise AssertionError("wavefront run mismatch")
            done += 1
            continue
        if mode == "shards":
            k = int(rng.integers(2, 5))
            b = g.partition(k)
            hs = [HyperBall(g, p, depth, node_range=(int(b[r]), int(b[r + 1]))) for r in range(k)]
        else:
            hs = [HyperBall(g, p, depth, skip_unchanged=(mode == "skip"), interval=(mode == "interval"),
                            schedule=sched)]
        t = 0
        while True:
            t += 1
            mx = max(h.step_compute() for h in hs)
            if len(hs) > 1:
                HyperBall.exchange_local(hs)
            fin = [h.step_finish(mx)[1] for h in hs][0]
            mo = O.hb_iterate(g, p, t, cur, nxt, c_prev, c_cur, sd, sd2)
            ok = mx == mo and np.array_equal(hs[0].registers(), nxt)
            ok &= np.array_equal(np.concatenate([h.state().sum_d for h in hs]), sd)
            ok &= np.array_equal(np.concatenate([h.state().c_curr for h in hs]), c_cur)
            if not ok:
                raise AssertionError(f"hyperball mismatch at t={t}")
            if fin != (mo <= 0.5 or (depth is not None and t == depth)):
                raise AssertionError("termination mismatch")
            if fin:
                break
            cur, nxt = nxt, cur
            c_prev, c_cur = c_cur, c_prev
        if case % 4 == 0 and not big:  # widened passes on every 4th graph
            lm, ref = DeviceGraph(g).local_metrics(), P.local_metrics(g)
            for key in ref:
                if not np.array_equal(lm[key], ref[key], equal_nan=lm[key].dtype.kind == "f"):
                    raise AssertionError(f"local metric {key}")
            ex, rx = exact_bfs_all(g, depth, interval=bool(rng.random() < 0.5)), P.exact_bfs(g, depth)
            for key in ("sum_d", "sum_d2", "reach"):
                if not np.array_equal(ex[key], rx[key]):
                    raise AssertionError(f"exact {key}")
        done += 1
    except Exception as e:  # record and continue
        fails.append(dict(params, error=f"{type(e).__name__}: {e}"))
print(json.dumps(dict(cases=done + len(fails), passed=done, failed=len(fails), oracle=O.kind,
                      seconds=time.time() - t_start, failures=fails[:20]), indent=1))

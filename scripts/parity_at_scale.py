"""Full-size parity: the GPU HyperBall vs the reference CPU path (the reference's
own compiled hll/kernels primitives + the SPEC loop, oracle/_ref) on a bench
config, compared after EVERY iteration: registers (reference packed layout,
SHA-256 + memcmp), c_t, sum_d, sum_d2 and the max increase.

usage: python scripts/parity_at_scale.py c2|c3 [p] [depth]
Prints one JSON object (per-iteration match flags, CPU and GPU seconds)."""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402  (parity checker: test infrastructure)
from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import HllParams, HyperBall  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 10
depth = int(sys.argv[3]) if len(sys.argv) > 3 and int(sys.argv[3]) > 0 else None
g = build_graph(cfg)
O = oracle.reference() if oracle.reference_available() else oracle.port()
threads = os.cpu_count() or 1
hb = HyperBall(g, HllParams(p), depth)
n = g.n
cur, c_prev = O.hb_init(n, p)
nxt = np.zeros_like(cur)
c_cur = np.zeros(n)
sd, sd2 = np.zeros(n), np.zeros(n)
rows, t, cpu_s, gpu_s = [], 0, 0.0, 0.0
ok_all = np.array_equal(hb.registers(), cur)
while True:
    t += 1
    t0 = time.perf_counter()
    mg = hb.iterate_once()
    gpu_s += time.perf_counter() - t0
    t0 = time.perf_counter()
    mo = O.hb_iterate(g, p, t, cur, nxt, c_prev, c_cur, sd, sd2, threads=threads)
    cpu_s += time.perf_counter() - t0
    regs = hb.registers()
    s = hb.state()
    row = dict(t=t, registers=bool(np.array_equal(regs, nxt)), c=bool(np.array_equal(s.c_curr, c_cur)),
               sum_d=bool(np.array_equal(s.sum_d, sd)), sum_d2=bool(np.array_equal(s.sum_d2, sd2)),
               max_increase=bool(mg == mo), max_increase_value=mo,
               registers_sha256=hashlib.sha256(nxt.tobytes()).hexdigest()[:16])
    rows.append(row)
    ok_all &= all(row[k] for k in ("registers", "c", "sum_d", "sum_d2", "max_increase"))
    fin = mo <= 0.5 or (depth is not None and t == depth)
    if fin:
        break
    cur, nxt = nxt, cur
    c_prev, c_cur = c_cur, c_prev
print(json.dumps(dict(config=cfg, p=p, depth=depth, nodes=n, edges=g.edges, oracle=O.kind, cpu_threads=threads,
                      iterations=t, all_bit_exact=bool(ok_all), cpu_seconds=cpu_s,
                      gpu_seconds_incl_readback=gpu_s, per_iteration=rows), indent=1))

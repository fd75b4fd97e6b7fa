"""Run-to-run determinism at C3: R full HyperBall runs per mode (dense tile
schedule, per-warp items and forced group schedules, skip-unchanged, interval, async upload, wavefront first run dense/interval), SHA-256
of the final registers and of sum_d must be identical across all runs and modes."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HyperBall  # noqa: E402

R = int(sys.argv[1]) if len(sys.argv) > 1 else 10
g = build_graph("c3")
dg = DeviceGraph(g)
hashes = {}
modes = {"dense": {}, "skip": {"skip_unchanged": True}, "interval": {"interval": True}}
for name, kw in modes.items():
    hb = HyperBall(dg, 10, None, **kw)
    hs = set()
    for _ in range(R):
        hb.reset()
        hb.run()
        hs.add((hashlib.sha256(hb.registers().tobytes()).hexdigest(),
                hashlib.sha256(hb.state().sum_d.tobytes()).hexdigest()))
    hashes[name] = sorted(hs)
    del hb
for sched in ("items", "group"):
    hb = HyperBall(dg, 10, None, schedule=sched)
    hb.run()
    hashes[f"dense_{sched}_schedule"] = [(hashlib.sha256(hb.registers().tobytes()).hexdigest(),
                                          hashlib.sha256(hb.state().sum_d.tobytes()).hexdigest())]
    del hb
hb = HyperBall(DeviceGraph(g, async_upload=True), 10, None)
hb.run()
hashes["async_upload"] = [(hashlib.sha256(hb.registers().tobytes()).hexdigest(),
                           hashlib.sha256(hb.state().sum_d.tobytes()).hexdigest())]
for name, kw in {"async_wavefront": {}, "async_wavefront_interval": {"interval": True}}.items():
    hb = HyperBall(DeviceGraph(g, async_upload=True), 10, None, wavefront=True, **kw)
    hb.run()
    hashes[name] = [(hashlib.sha256(hb.registers().tobytes()).hexdigest(),
                     hashlib.sha256(hb.state().sum_d.tobytes()).hexdigest())]
    del hb
distinct = {h for v in hashes.values() for h in v}
print(json.dumps(dict(runs_per_mode=R, modes=list(hashes), distinct_results=len(distinct),
                      deterministic=len(distinct) == 1, hash=sorted(distinct)[0]), indent=1))

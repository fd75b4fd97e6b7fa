"""Per-iteration host/launch overhead: step_ms (wall, incl. sync) minus the kernel times."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import HyperBall  # noqa: E402

out = {}
for cfg in ("c1", "c2"):
    g = build_graph(cfg)
    for interval in (False, True):
        h = HyperBall(g, 10, None, interval=interval)
        for _ in range(3):
            h.reset()
            h.run()
        st = h.stats()
        step = np.array([s["step_ms"] for s in st])
        kern = np.array([s["union_ms"] + s["estimate_ms"] for s in st])
        out[f"{cfg}_{'interval' if interval else 'dense'}"] = dict(
            iterations=len(st), step_ms=float(step.mean()), kernels_ms=float(kern.mean()),
            overhead_ms=float((step - kern).mean()))
print(json.dumps(out, indent=1))

#!/usr/bin/env python
"""Dense union ms/iteration per schedule (auto / group / items) at p = 6..10 on
C1 and C2 (and C3 at p = 8, 9): evidence for the precision at which the
16-node group path takes over from per-node work items (sb_hb_api.cu)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph, HllParams, HyperBall  # noqa: E402
from scripts.sweep import time_runs  # noqa: E402


def main():
    torch.cuda.set_device(0)
    out = []
    for cfg, ps in (("c1", (4, 6, 8, 10)), ("c2", (4, 5, 6, 7, 8, 9, 10)), ("c3", (8, 9))):
        g = build_graph(cfg)
        dg = DeviceGraph(g, 0)
        for p in ps:
            row = {"config": cfg, "p": p}
            for sched in ("auto", "group", "items"):
                hb = HyperBall(dg, HllParams(p), 3 if cfg == "c1" else None, schedule=sched)
                it, sec, ums = time_runs(hb)
                row[sched] = round(ums, 4)
                del hb
            print(json.dumps(row), flush=True)
            out.append(row)
        del dg
    json.dump(out, open(os.path.join(ROOT, "gpurun_out", "group_threshold.json"), "w"), indent=1)


if __name__ == "__main__":
    main()

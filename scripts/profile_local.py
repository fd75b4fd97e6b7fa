"""Local-metrics pass on a C3 node sub-range (for ncu): python scripts/profile_local.py [v0] [count]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import DeviceGraph  # noqa: E402

v0 = int(sys.argv[1]) if len(sys.argv) > 1 else 117000
cnt = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
g = build_graph("c3")
dg = DeviceGraph(g)
dg.local_metrics(v0, v0 + 8)
m = dg.local_metrics(v0, v0 + cnt)
print("mean n2", float(m["n2"].mean()))

#!/usr/bin/env python
"""Per-phase cycle shares of the dense union's group path on one graph, from the
instrumented build (`make stats`; SB_LIBRARY points the package at it).

  SB_LIBRARY=paper_2604_08374_b200/libsieveball_cuda_stats.so python scripts/group_stats.py [c3|c2|c1] [p]

Cycles are summed over warps (clock64 laps), so the shares say where a warp's
time goes, barrier waits included; the instrumented kernel is slower than the
product one, so only the proportions and the work counts are meaningful."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import build_graph  # noqa: E402
from paper_2604_08374_b200 import HyperBall  # noqa: E402
from paper_2604_08374_b200._lib import lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
p = int(sys.argv[2]) if len(sys.argv) > 2 else 10
g = build_graph(cfg)
hb = HyperBall(g, p, 1)
L = lib()
f = L.sb_debug_group_stats
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
buf = (C.c_ulonglong * 16)()
hb.run()
f(buf, 1)  # reset after the warm-up pass
hb.reset()
hb.run()   # one union pass (depth 1)
f(buf, 0)
st = list(buf)
names = {8: "A decode->bitmaps", 9: "barrier 1 wait", 10: "B0 block ANDs", 11: "barrier 2 wait",
         12: "B1 folds (blocks, root slices)", 13: "(unused)", 14: "barrier 3 wait", 15: "end of group"}
tot = sum(st[i] for i in names)
print(f"{cfg} p={p}: groups={st[5] // 8} windows={st[0] // 8} windows/group={st[0] / max(st[5], 1):.2f} "
      f"decode steps={st[1]} root rows={st[2]} block rows={st[3]} block passes={st[4]}")
print(f"decode steps per window per node={st[1] / max(st[0] / 8, 1) / 16:.2f}  rows per group: root="
      f"{st[2] / max(st[5] / 8, 1):.0f} blocks={st[3] / max(st[5] / 8, 1):.0f}")
for i, n in names.items():
    print(f"  {n:22s} {100 * st[i] / tot:5.1f} %")

"""Paper Table 1 analogue: HyperBall (p = 8/10/12) vs the exact GPU BFS on five
synthetic towns; prints one JSON object (rows + per-precision means)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from tests.test_exact import accuracy_table  # noqa: E402

tab = accuracy_table((8, 10, 12, 14))
means = {p: dict(md_err=float(np.mean([r["md_err"] for r in tab if r["p"] == p])),
                 md_r=float(np.mean([r["md_r"] for r in tab if r["p"] == p])),
                 ihh_rho=float(np.mean([r["ihh_rho"] for r in tab if r["p"] == p]))) for p in (8, 10, 12, 14)}
print(json.dumps(dict(rows=tab, means=means), indent=1))

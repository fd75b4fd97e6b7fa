"""compare(estimate, exact) -- the oracle module's accuracy report.

Pearson r over nodes finite in both inputs, Spearman rho with average ranks
for ties, median relative error; one row per metric.  Used by cmd_validate and
by the paper Table 1 analogue (acceptance criterion 4: HyperBall at p=10 vs
the exact BFS).
"""
from __future__ import annotations

import csv

import numpy as np


def _rank(x: np.ndarray) -> np.ndarray:
    order = np.argsort(x, kind="mergesort")
    r = np.empty(len(x), np.float64)
    xs = x[order]
    i = 0
    while i < len(xs):  # average ranks over ties
        j = i
        while j + 1 < len(xs) and xs[j + 1] == xs[i]:
            j += 1
        r[order[i:j + 1]] = 0.5 * (i + j) + 1.0
        i = j + 1
    return r


def pearson(a: np.ndarray, b: np.ndarray) -> float:
    a = a - a.mean()
    b = b - b.mean()
    den = np.sqrt((a * a).sum() * (b * b).sum())
    return float((a * b).sum() / den) if den > 0 else (1.0 if np.array_equal(a, b) else float("nan"))


def spearman(a: np.ndarray, b: np.ndarray) -> float:
    return pearson(_rank(a), _rank(b))


def compare(estimate: dict[str, np.ndarray], exact: dict[str, np.ndarray],
            metrics=("md", "ihh", "tekl", "pv")) -> list[dict]:
    rows = []
    for k in metrics:
        if k not in estimate or k not in exact:
            continue
        e, x = np.asarray(estimate[k], np.float64), np.asarray(exact[k], np.float64)
        if e.shape != x.shape:
            raise ValueError(f"compare: node sets differ for {k}")
        ok = np.isfinite(e) & np.isfinite(x)
        e, x = e[ok], x[ok]
        nz = x != 0
        rel = np.abs(e[nz] - x[nz]) / np.abs(x[nz])
        rows.append(dict(metric=k, pearson_r=pearson(e, x) if e.size > 1 else float("nan"),
                         spearman_rho=spearman(e, x) if e.size > 1 else float("nan"),
                         median_rel_err=float(np.median(rel)) if rel.size else float("nan"), n=int(e.size)))
    return rows


def write_report(path: str, rows: list[dict]) -> None:
    """CSV: metric, pearson_r, spearman_rho, median_rel_err, n."""
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=["metric", "pearson_r", "spearman_rho", "median_rel_err", "n"])
        w.writeheader()
        for r in rows:
            w.writerow(r)

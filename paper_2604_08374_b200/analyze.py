"""cmd_analyze: graph -> per-node MetricRow table -> CSV.

mode "hyperball": HyperBall on the GPU (HLL precision p, depth limit d), the
BFS metrics from its sums (sb_hb_metrics), entropy columns NaN.
mode "exact": the exact bit-parallel BFS on the GPU (sb_exact_*), metrics
from the exact sums, entropy from the depth histogram.  Both modes add the
exact local metrics (sb_local_metrics) -- bit-equal between modes
(acceptance criterion 9) because they never touch the HLL state.
"""
from __future__ import annotations

import ctypes as C
import time

import numpy as np

from ._lib import check, lib, sb_metric_table
from .cgraph import CompressedCsr
from .exact import ExactBfs
from .hyperball import DeviceGraph, HllParams, HyperBall
from . import metrics as M

COLUMNS = ("x", "y", "node_id", "component_id", "node_count", "connectivity", "visual_mean_depth",
           "integration_hh", "integration_tekl", "integration_pv", "control", "controllability", "clustering",
           "entropy", "rel_entropy", "first_moment", "second_moment")


def metrics_from_sums(sum_d: np.ndarray, sum_d2: np.ndarray, nv: np.ndarray, deg: np.ndarray) -> dict:
    """MD / IHH / Tekl / PV / moments from (exact) depth sums, SPEC.md:485-529 closed forms."""
    f = np.vectorize
    sd = np.asarray(sum_d, np.float64)
    sd2 = np.asarray(sum_d2, np.float64)
    nvi = np.asarray(nv, np.int64)
    md = f(M.mean_depth, otypes=[float])(sd, nvi) if sd.size else np.zeros(0)
    ihh = f(M.integration_hh, otypes=[float])(md, nvi) if sd.size else np.zeros(0)
    tekl = np.where(nvi >= 2, np.log2((md + 2.0) / 3.0), np.nan) if sd.size else np.zeros(0)
    pv = f(M.integration_pv, otypes=[float])(md, nvi) if sd.size else np.zeros(0)
    m1 = np.where(nvi >= 2, md * np.asarray(deg, np.float64), np.nan)
    m2 = np.where(nvi >= 2, sd2 / np.maximum(nvi - 1.0, 1.0), np.nan)
    return dict(md=md, ihh=ihh, tekl=tekl, pv=pv, m1=m1, m2=m2)


def analyze(csr: CompressedCsr, p: int = 10, depth_limit: int | None = None, mode: str = "hyperball",
            out: str | None = None, device: int = 0, interval: bool = False, local: bool = True) -> dict:
    """Runs the pipeline on one GPU; returns the columns (+ timings); writes CSV to `out`."""
    if mode not in ("hyperball", "exact"):
        raise ValueError("mode must be 'hyperball' or 'exact'")
    HllParams(p)  # validates p in both modes
    timings = {}
    t0 = time.perf_counter()
    dg = DeviceGraph(csr, device)
    timings["upload_s"] = time.perf_counter() - t0
    nv = np.ascontiguousarray(csr.node_count_of_component(), np.uint32)
    deg = np.ascontiguousarray(csr.degrees, np.uint32)
    t0 = time.perf_counter()
    if mode == "hyperball":
        hb = HyperBall(dg, p, depth_limit, interval=interval)
        iterations = hb.run()
        m = hb.metrics(nv, deg)
        entropy = np.full(csr.n, np.nan)
    else:
        x = ExactBfs(dg, depth_limit, interval=interval)
        x.run()
        r = x.result()
        iterations = x.stats()["max_depth"]
        m = metrics_from_sums(r["sum_d"], r["sum_d2"], nv, deg)
        entropy = r["entropy"]
    timings["bfs_s"] = time.perf_counter() - t0
    cols = dict(md=m["md"], ihh=m["ihh"], tekl=m["tekl"], pv=m["pv"], m1=m["m1"], m2=m["m2"], entropy=entropy,
                rel_entropy=np.full(csr.n, np.nan))
    if local:
        t0 = time.perf_counter()
        lm = dg.local_metrics()
        timings["local_s"] = time.perf_counter() - t0
        cols.update(control=lm["control"], controllability=lm["controllability"], clustering=lm["clustering"])
    x, y = csr.coordinates()
    # node_id is the ORIGINAL id: a Hilbert-reordered graph maps each row back
    # through hilbert_inverse, otherwise the row index.
    node_id = csr.hilbert_inverse if csr.hilbert_inverse is not None else np.arange(csr.n, dtype=np.uint32)
    cols.update(x=np.ascontiguousarray(x, np.float64), y=np.ascontiguousarray(y, np.float64),
                node_id=np.ascontiguousarray(node_id, np.uint32), component_id=np.ascontiguousarray(csr.component_id, np.uint32), node_count=nv, connectivity=deg)
    if out is not None:
        t0 = time.perf_counter()
        write_csv(out, cols, csr.n)
        timings["write_s"] = time.perf_counter() - t0
    cols["iterations"] = iterations
    cols["timings"] = timings
    return cols


def write_csv(path: str, cols: dict, n: int) -> None:
    """sb_metrics_write_csv over whichever columns are present (missing -> NaN)."""
    keep = {}
    t = sb_metric_table()
    t.n = n

    def put(field, key, dtype):
        if key in cols and cols[key] is not None:
            a = np.ascontiguousarray(cols[key], dtype)
            assert a.size == n, key
            keep[field] = a
            setattr(t, field, a.ctypes.data)

    for field, key in (("x", "x"), ("y", "y"), ("md", "md"), ("ihh", "ihh"), ("tekl", "tekl"), ("pv", "pv"),
                       ("control", "control"), ("controllability", "controllability"), ("clustering", "clustering"),
                       ("entropy", "entropy"), ("rel_entropy", "rel_entropy"), ("m1", "m1"), ("m2", "m2")):
        put(field, key, np.float64)
    for field in ("node_id", "component_id", "node_count", "connectivity"):
        put(field, field, np.uint32)
    check(lib().sb_metrics_write_csv(path.encode(), C.byref(t)))


BENCH_HEADER = ("depth", "iterations", "last_changing_pass", "bfs_seconds", "union_ms", "mean_md", "max_increase")


def bench_depths(csr: CompressedCsr, depths=(3, 5, 10, None), p: int = 10, out: str | None = None,
                 device: int = 0, interval: bool = False) -> list[dict]:
    """cmd_bench (paper Table 3 shape): one HyperBall run per depth limit
    (None = unlimited) -> depth, iterations, BFS time (device, summed per-iteration
    kernel + exchange time), mean MD as the accuracy proxy; optional CSV."""
    dg = DeviceGraph(csr, device)
    nv = np.ascontiguousarray(csr.node_count_of_component(), np.uint32)
    deg = np.ascontiguousarray(csr.degrees, np.uint32)
    rows = []
    for d in depths:
        hb = HyperBall(dg, p, d, interval=interval)
        hb.run()  # warm
        hb.reset()
        it = hb.run()
        st = hb.stats()
        m = hb.metrics(nv, deg)
        rows.append(dict(depth="unlimited" if d is None else int(d), iterations=it,
                         last_changing_pass=max([s["t"] for s in st if s["changed_nodes"] > 0], default=0),
                         bfs_seconds=sum(s["step_ms"] for s in st) / 1e3,
                         union_ms=sum(s["union_ms"] for s in st), mean_md=float(np.nanmean(m["md"])),
                         max_increase=st[-1]["max_increase"] if st else 0.0))
    if out is not None:
        import csv
        with open(out, "w", newline="") as f:
            w = csv.DictWriter(f, fieldnames=list(BENCH_HEADER))
            w.writeheader()
            for r in rows:
                w.writerow(r)
    return rows


def validate_graph(csr: CompressedCsr, p: int = 10, depth_limit: int | None = None, out: str | None = None,
                   device: int = 0) -> list[dict]:
    """cmd_validate: both modes on the same graph, compare() report
    (Pearson r, Spearman rho, median relative error per metric)."""
    from . import validate
    hb = analyze(csr, p, depth_limit, "hyperball", device=device, local=False)
    ex = analyze(csr, p, depth_limit, "exact", device=device, local=False)
    rows = validate.compare(hb, ex)
    if out is not None:
        validate.write_report(out, rows)
    return rows

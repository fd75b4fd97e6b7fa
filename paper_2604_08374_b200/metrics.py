"""VGA metrics from HyperBall sums, scalar closed forms.

The per-node batch runs on the device (HyperBall.metrics -> sb_hb_metrics);
these scalar forms mirror the SPEC operations one-to-one for host callers.
"""
from __future__ import annotations

import math


def mean_depth(sum_d: float, n_v: int) -> float:
    """MD = sum_d / (N_v - 1); NaN for N_v < 2."""
    return float("nan") if n_v < 2 else sum_d / (n_v - 1.0)


def relative_asymmetry(md: float, n_v: int) -> float:
    return 2.0 * (md - 1.0) / (n_v - 2.0)


def diamond(k: float) -> float:
    """D_k = 2(k(log2((k+2)/3) - 1) + 1) / ((k-1)(k-2))."""
    return 2.0 * (k * (math.log2((k + 2.0) / 3.0) - 1.0) + 1.0) / ((k - 1.0) * (k - 2.0))


def integration_hh(md: float, n_v: int) -> float:
    """1 / RRA; NaN unless N_v >= 3 and MD > 1."""
    if n_v < 3 or math.isnan(md) or not md > 1.0:
        return float("nan")
    return 1.0 / (relative_asymmetry(md, n_v) / diamond(n_v))


def integration_tekl(md: float) -> float:
    """log2((MD+2)/3)."""
    return math.log2((md + 2.0) / 3.0)


def integration_pv(md: float, n_v: int) -> float:
    """max(0, 1 - RA), clamped to [0, 1]: an HLL
    estimate can put MD below 1."""
    if n_v < 3 or math.isnan(md):
        return float("nan")
    return min(1.0, max(0.0, 1.0 - relative_asymmetry(md, n_v)))


def moments(md: float, deg: int, sum_d2: float, n_v: int) -> tuple[float, float]:
    """(MD * deg, sum_d2 / (N_v - 1))."""
    if n_v < 2:
        return float("nan"), float("nan")
    return md * deg, sum_d2 / (n_v - 1.0)

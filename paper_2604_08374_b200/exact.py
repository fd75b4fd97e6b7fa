"""Exact mode: the reference oracle's exact BFS / neighbourhood function on the GPU.

SPEC.md:583-606 (`exact_bfs_all`, ExactResult) computes per-source BFS on the
CPU.  Here it is the HyperBall loop with every HLL row replaced by an exact
reachability bitset over a block of 2^log2_block sources and the register max
replaced by OR (sb_exact_* in libsieveball_cuda.so) -- the same fused
decode-union kernel, bit-parallel over sources.  Sources shard freely across
GPUs (sum the outputs); there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import SB_HB_INTERVAL, check, lib, ptr
from .cgraph import CompressedCsr
from .hyperball import DeviceGraph


class ExactBfs:
    """exact_bfs_all(graph, depth_limit) over a source range."""

    def __init__(self, graph: CompressedCsr | DeviceGraph, depth_limit: int | None = None, log2_block: int = 12,
                 interval: bool = False, device: int = 0):
        self.graph = graph if isinstance(graph, DeviceGraph) else DeviceGraph(graph, device)
        self.depth_limit = depth_limit
        self._h = C.c_void_p()
        check(lib().sb_exact_create(self.graph._h, int(log2_block), int(depth_limit or 0),
                                    SB_HB_INTERVAL if interval else 0, C.byref(self._h)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sb_exact_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def run(self, src_begin: int = 0, src_end: int | None = None) -> int:
        """Accumulates BFS from sources [src_begin, src_end); returns the max depth seen so far."""
        src_end = self.graph.n if src_end is None else src_end
        md = C.c_uint32()
        check(lib().sb_exact_run(self._h, src_begin, src_end, C.byref(md)))
        return md.value

    def stats(self) -> dict:
        s, md, ms, nl = C.c_uint64(), C.c_uint32(), C.c_double(), C.c_uint64()
        check(lib().sb_exact_stats(self._h, C.byref(s), C.byref(md), C.byref(ms), C.byref(nl)))
        return dict(sources_done=s.value, max_depth=md.value, union_ms=ms.value, union_launches=nl.value)

    def result(self, with_hist: bool = True) -> dict[str, np.ndarray]:
        """ExactResult: sum_d, sum_d2, reach, depth histogram, entropy."""
        n = self.graph.n
        sd, sd2 = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        reach = np.zeros(n, np.uint32)
        out = dict(sum_d=sd, sum_d2=sd2, reach=reach)
        hist = None
        if with_hist:
            cap = self.stats()["max_depth"] + 1
            hist = np.zeros(n * cap, np.uint32)
            out["hist"] = hist.reshape(n, cap)
        check(lib().sb_exact_read(self._h, ptr(sd), ptr(sd2), ptr(reach), ptr(hist), out["hist"].shape[1]
                                  if with_hist else 0))
        if with_hist:
            out["entropy"] = depth_entropy(out["hist"])
        return out


def depth_entropy(hist: np.ndarray) -> np.ndarray:
    """Shannon entropy (bits) of each node's depth distribution (sb_depth_entropy)."""
    h = np.ascontiguousarray(hist, np.uint32)
    n, cap = h.shape
    ent = np.zeros(n, np.float64)
    check(lib().sb_depth_entropy(n, ptr(h), cap, ptr(ent)))
    return ent


def neighbourhood_function(hist: np.ndarray) -> np.ndarray:
    """|B(v, t)| for t = 0..D: 1 + cumulative depth counts."""
    b = np.cumsum(hist.astype(np.int64), axis=1)
    return b - hist[:, :1] + 1


def exact_bfs_all(graph: CompressedCsr, depth_limit: int | None = None, interval: bool = False,
                  device: int = 0) -> dict[str, np.ndarray]:
    x = ExactBfs(graph, depth_limit, interval=interval, device=device)
    x.run()
    r = x.result()
    r["stats"] = x.stats()
    return r

"""sieveball-b200: B200-native HyperBall hot path of arxiv 2604.08374.

Drop-in for the reference's HyperBall path (compressed-CSR loader, HyperBall
runner, VGA metrics).  Host API mirrors SPEC.md's hyperball / cgraph / hll /
metrics modules; compute runs in libsieveball_cuda.so (sm_100a).
"""
from ._lib import CudaError, NcclError, lib  # noqa: F401
from .cgraph import CompressedCsr, encode_neighbor_row, grid_mask, leb128_decode, leb128_encode  # noqa: F401
from .hyperball import (Comm, DeviceGraph, HllParams, HyperBall, HyperBallState,  # noqa: F401
                        check_convergence, release_cached_memory, run)
from . import metrics  # noqa: F401
from .exact import ExactBfs, depth_entropy, exact_bfs_all, neighbourhood_function  # noqa: F401
from .analyze import analyze, bench_depths, metrics_from_sums, validate_graph, write_csv  # noqa: F401
from . import validate  # noqa: F401

__all__ = ["CompressedCsr", "DeviceGraph", "HllParams", "HyperBall", "HyperBallState", "Comm",
           "check_convergence", "release_cached_memory", "run", "metrics", "leb128_encode", "leb128_decode",
           "encode_neighbor_row", "lib", "ExactBfs",
           "exact_bfs_all", "depth_entropy", "neighbourhood_function", "analyze", "metrics_from_sums", "write_csv",
           "validate", "grid_mask", "bench_depths", "validate_graph"]

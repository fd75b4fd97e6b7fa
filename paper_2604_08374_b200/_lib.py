"""ctypes binding of libsieveball_cuda.so (the C-ABI in include/sieveball_cuda.h).

The library is built in-tree (``make`` / ``__graft_entry__.build()``).  There
is no fallback: importing the package without the shared object raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsieveball_cuda.so")

SB_OK, SB_EINVAL, SB_ERUNTIME, SB_ECUDA, SB_ENCCL, SB_ENOMEM = range(6)
SB_HB_SKIP_UNCHANGED = 1
SB_HB_SCHEDULE_WARP = 2
SB_HB_INTERVAL = 4
SB_HB_SCHEDULE_GROUP = 8
SB_HB_WAVEFRONT = 16
SB_REGS_LATEST, SB_REGS_PREVIOUS = 0, 1
SB_COMM_ID_BYTES = 128
SB_IPC_HANDLE_BYTES = 256


class CudaError(RuntimeError):
    """A CUDA runtime failure (SB_ECUDA)."""


class NcclError(RuntimeError):
    """An NCCL failure (SB_ENCCL)."""


class sb_csr_desc(C.Structure):
    _fields_ = [
        ("n", C.c_uint64), ("edges", C.c_uint64), ("stream_len", C.c_uint64),
        ("offsets", C.POINTER(C.c_uint64)), ("degrees", C.POINTER(C.c_uint32)),
        ("stream", C.POINTER(C.c_uint8)), ("n_components", C.c_uint64),
        ("component_id", C.POINTER(C.c_uint32)), ("component_sizes", C.POINTER(C.c_uint32)),
        ("cell_of_node", C.POINTER(C.c_uint32)), ("hilbert_inverse", C.POINTER(C.c_uint32)),
        ("origin_x", C.c_double), ("origin_y", C.c_double), ("spacing", C.c_double),
        ("rows", C.c_uint32), ("cols", C.c_uint32),
    ]


class sb_iter_stats(C.Structure):
    _fields_ = [
        ("t", C.c_uint32), ("union_ms", C.c_float), ("estimate_ms", C.c_float),
        ("exchange_ms", C.c_float), ("step_ms", C.c_float), ("max_increase", C.c_double),
        ("changed_nodes", C.c_uint64),
    ]


class sb_metric_table(C.Structure):
    _fields_ = [("n", C.c_uint64), ("node_id", C.c_void_p), ("x", C.c_void_p), ("y", C.c_void_p),
                ("component_id", C.c_void_p), ("node_count", C.c_void_p), ("connectivity", C.c_void_p)] + [
        (k, C.c_void_p) for k in ("md", "ihh", "tekl", "pv", "control", "controllability", "clustering",
                                  "entropy", "rel_entropy", "m1", "m2")]


_vp = C.c_void_p
_u64 = C.c_uint64
_u32 = C.c_uint32
_i = C.c_int
_pp = C.POINTER(C.c_void_p)

# name -> (restype, argtypes)
_SIGS = {
    "sb_last_error": (C.c_char_p, []),
    "sb_version": (C.c_char_p, []),
    "sb_device_count": (_i, [C.POINTER(_i)]),
    "sb_release_cached_memory": (_i, [_i]),
    "sb_check_convergence": (_i, [C.c_double]),
    "sb_csr_synth_grid": (_i, [_u32, _u32, _u32, _u32, _u32, _u64, _u64, C.c_uint, _pp]),
    "sb_csr_from_adjacency": (_i, [_u64, _vp, _vp, _pp]),
    "sb_csr_from_arrays": (_i, [_u64, _vp, _vp, _vp, _u64, _pp]),
    "sb_csr_describe": (_i, [_vp, C.POINTER(sb_csr_desc)]),
    "sb_csr_neighbors": (_i, [_vp, _u64, _vp]),
    "sb_csr_hilbert_reorder": (_i, [_vp, _pp]),
    "sb_vgacsr_save": (_i, [_vp, C.c_char_p]),
    "sb_vgacsr_load": (_i, [C.c_char_p, _pp]),
    "sb_csr_destroy": (None, [_vp]),
    "sb_csr_pin": (_i, [_vp, _i]),
    "sb_partition_edges": (_i, [_u64, _vp, _vp, _i, _vp]),
    "sb_graph_create": (_i, [_u64, _vp, _vp, _vp, _u64, _vp, _u64, _u64, _i, _pp]),
    "sb_graph_stats": (_i, [_vp, C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u64), C.POINTER(_u32)]),
    "sb_graph_destroy": (None, [_vp]),
    "sb_graph_create_async": (_i, [_u64, _vp, _vp, _vp, _u64, _vp, _u64, _u64, _i, _pp]),
    "sb_graph_wait": (_i, [_vp]),
    "sb_graph_build_grid": (_i, [_u32, _u32, _vp, _u64, _i, _pp]),
    "sb_graph_grid_info": (_i, [_vp, C.POINTER(_u32), C.POINTER(_u32), _vp, _vp, _vp, C.POINTER(_u64)]),
    "sb_graph_download": (_i, [_vp, _vp, _vp, _vp]),
    "sb_grid_synth_mask": (_i, [_u32, _u32, _u32, _u32, _u32, _u64, _vp]),
    "sb_hb_create": (_i, [_vp, C.c_uint, _u32, _u32, _pp]),
    "sb_hb_step": (_i, [_vp, C.POINTER(C.c_double), C.POINTER(_i), C.POINTER(_i)]),
    "sb_hb_run": (_i, [_vp, C.POINTER(_u32), C.POINTER(_i)]),
    "sb_hb_step_compute": (_i, [_vp, C.POINTER(C.c_double)]),
    "sb_hb_exchange_local": (_i, [C.POINTER(_vp), _i]),
    "sb_hb_step_finish": (_i, [_vp, C.c_double, C.POINTER(_i), C.POINTER(_i)]),
    "sb_hb_read_registers": (_i, [_vp, _i, _u64, _u64, _vp]),
    "sb_hb_set_registers": (_i, [_vp, _vp]),
    "sb_hb_read_state": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, C.POINTER(_u32), C.POINTER(_i), C.POINTER(_i)]),
    "sb_hb_metrics": (_i, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "sb_local_metrics": (_i, [_vp, _u64, _u64, _vp, _vp, _vp, _vp, _vp]),
    "sb_exact_create": (_i, [_vp, C.c_uint, _u32, _u32, _pp]),
    "sb_exact_run": (_i, [_vp, _u64, _u64, C.POINTER(_u32)]),
    "sb_exact_read": (_i, [_vp, _vp, _vp, _vp, _vp, _u32]),
    "sb_exact_stats": (_i, [_vp, C.POINTER(_u64), C.POINTER(_u32), C.POINTER(C.c_double), C.POINTER(_u64)]),
    "sb_exact_destroy": (None, [_vp]),
    "sb_depth_entropy": (_i, [_u64, _vp, _u32, _vp]),
    "sb_metrics_write_csv": (_i, [C.c_char_p, C.POINTER(sb_metric_table)]),
    "sb_hb_stats": (_i, [_vp, C.POINTER(sb_iter_stats), _u32, C.POINTER(_u32)]),
    "sb_hb_reset": (_i, [_vp]),
    "sb_hb_stream": (_vp, [_vp]),
    "sb_hb_destroy": (None, [_vp]),
    "sb_comm_unique_id": (_i, [_vp]),
    "sb_comm_create": (_i, [_i, _i, _vp, _i, _pp]),
    "sb_hb_attach_comm": (_i, [_vp, _vp, _vp]),
    "sb_comm_destroy": (None, [_vp]),
    "sb_hb_ipc_handles": (_i, [_vp, _vp, C.c_size_t]),
    "sb_hb_attach_peers": (_i, [_vp, _i, _i, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def _preload_torch_nccl() -> None:
    """Load the NCCL that torch ships (the nvidia-nccl wheel) before this library, so
    both bind one libnccl.so.2 whichever is imported first.  Otherwise loading this
    library first binds the system NCCL and a later `import torch` fails on symbols
    only the wheel's newer NCCL has."""
    try:
        import nvidia.nccl as nn
    except ImportError:
        return
    for d in getattr(nn, "__path__", []):
        so = os.path.join(d, "lib", "libnccl.so.2")
        if os.path.exists(so):
            C.CDLL(so, mode=C.RTLD_GLOBAL)
            return


def lib() -> C.CDLL:
    """Load the in-tree shared object (fails loudly if it was not built).
    SB_LIBRARY may name another build of the same sources (the instrumented
    `make stats` build used by scripts/group_stats.py)."""
    global _lib
    if _lib is None:
        path = os.environ.get("SB_LIBRARY", LIB_PATH)
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `make` or __graft_entry__.build(); "
                "the HyperBall path has no CPU fallback")
        _preload_torch_nccl()
        L = C.CDLL(path)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a C-ABI return code onto the reference's exception classes."""
    if rc == SB_OK:
        return
    msg = lib().sb_last_error().decode(errors="replace")
    if rc == SB_EINVAL:
        raise ValueError(msg)  # std::invalid_argument
    if rc == SB_ECUDA:
        raise CudaError(msg)
    if rc == SB_ENCCL:
        raise NcclError(msg)
    if rc == SB_ENOMEM:
        raise MemoryError(msg)
    raise RuntimeError(msg)  # std::runtime_error


def ptr(a) -> int | None:
    """Raw data pointer of a contiguous numpy array (None for None)."""
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "array must be C-contiguous"
    return a.ctypes.data

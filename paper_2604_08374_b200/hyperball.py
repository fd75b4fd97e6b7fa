"""HyperBall on B200 -- Python mirror of the reference's hyperball module.

Names, argument meaning and error behaviour follow SPEC.md:407-472:
``run(graph, params, depth_limit)``, ``iterate_once``, ``check_convergence``,
``HllParams(p)`` raising ValueError (std::invalid_argument, hll.cpp:10) and
RuntimeError for malformed graphs (std::runtime_error, leb128.hpp:32,38).
Everything executes on the GPU through libsieveball_cuda.so; there is no CPU
fallback.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (SB_COMM_ID_BYTES, SB_HB_INTERVAL, SB_HB_SCHEDULE_GROUP, SB_HB_SCHEDULE_WARP, SB_HB_WAVEFRONT,
                   SB_HB_SKIP_UNCHANGED, SB_IPC_HANDLE_BYTES, SB_REGS_LATEST, SB_REGS_PREVIOUS, check, lib, ptr, sb_iter_stats)
from .cgraph import CompressedCsr


class HllParams:
    """HllParams (hll.hpp:22-29, hll.cpp:9-19)."""

    def __init__(self, precision: int):
        p = int(precision)
        if p < 4 or p > 16:
            raise ValueError("hll: precision must be in [4, 16]")
        self.p = p
        self.m = 1 << p
        self.row_bytes = self.m // 2
        self.alpha_m = {16: 0.673, 32: 0.697, 64: 0.709}.get(self.m, 0.7213 / (1.0 + 1.079 / self.m))

    def __repr__(self) -> str:
        return f"HllParams(p={self.p})"


def release_cached_memory(device: int = 0) -> None:
    """Return the device memory cached by freed graphs / HyperBall states to the driver."""
    check(lib().sb_release_cached_memory(device))


def check_convergence(max_increase: float) -> bool:
    """True iff max_increase <= 0.5 (inclusive)."""
    return bool(lib().sb_check_convergence(float(max_increase)))


@dataclass
class HyperBallState:
    """SPEC.md:412-415 (local node range)."""
    registers: np.ndarray | None
    c_prev: np.ndarray
    c_curr: np.ndarray
    sum_d: np.ndarray
    sum_d2: np.ndarray
    changed: np.ndarray
    t: int
    converged: bool
    finished: bool
    stats: list = field(default_factory=list)


class Comm:
    """NCCL communicator for node-range sharding (one process per GPU)."""

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(SB_COMM_ID_BYTES)
        check(lib().sb_comm_unique_id(buf))
        return buf.raw

    def __init__(self, nranks: int, rank: int, uid: bytes, device: int):
        assert len(uid) == SB_COMM_ID_BYTES
        self._h = C.c_void_p()
        check(lib().sb_comm_create(nranks, rank, uid, device, C.byref(self._h)))
        self.nranks, self.rank, self.device = nranks, rank, device

    def close(self):
        if self._h is not None and self._h.value:
            lib().sb_comm_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


class DeviceGraph:
    """Rows [v0, v1) of a CompressedCsr resident in HBM (validated at upload)."""

    def __init__(self, csr: CompressedCsr, device: int = 0, node_range: tuple[int, int] | None = None,
                 orig_id: np.ndarray | None = None, async_upload: bool = False):
        """async_upload: chunked upload overlapped with the first HyperBall pass
        (sb_graph_create_async); `csr` must stay alive until wait() / the first step."""
        v0, v1 = node_range if node_range is not None else (0, csr.n)
        oid = orig_id if orig_id is not None else csr.hilbert_inverse
        oid = None if oid is None else np.ascontiguousarray(oid, np.uint32)
        self._h = C.c_void_p()
        self._csr = csr if async_upload else None  # keeps the host stream alive during the upload
        fn = lib().sb_graph_create_async if async_upload else lib().sb_graph_create
        check(fn(csr.n, ptr(csr.offsets), ptr(csr.degrees), ptr(csr.stream_padded()), csr.stream_len, ptr(oid),
                 v0, v1, device, C.byref(self._h)))
        self.n, self.v0, self.v1, self.device = csr.n, v0, v1, device
        nl, el, sl, ni = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        ch = C.c_uint32()
        check(lib().sb_graph_stats(self._h, C.byref(nl), C.byref(el), C.byref(sl), C.byref(ni), C.byref(ch)))
        self.n_local, self.edges_local, self.stream_bytes_local = nl.value, el.value, sl.value
        self.n_items, self.chunk = ni.value, ch.value

    @classmethod
    def from_grid(cls, blocked: np.ndarray, radius2: int = 0, device: int = 0) -> "DeviceGraph":
        """Builds the grid visibility graph ON THE DEVICE (sb_graph_build_grid): blocked is a
        (rows, cols) mask of obstacle cells; radius2 in cells^2 (0 = unlimited)."""
        m = np.ascontiguousarray(blocked, np.uint8)
        if m.ndim != 2:
            raise ValueError("blocked must be a 2-D (rows, cols) mask")
        self = cls.__new__(cls)
        self._h = C.c_void_p()
        check(lib().sb_graph_build_grid(m.shape[0], m.shape[1], ptr(m), int(radius2), device, C.byref(self._h)))
        nl, el, sl, ni = C.c_uint64(), C.c_uint64(), C.c_uint64(), C.c_uint64()
        ch = C.c_uint32()
        check(lib().sb_graph_stats(self._h, C.byref(nl), C.byref(el), C.byref(sl), C.byref(ni), C.byref(ch)))
        self.n, self.v0, self.v1, self.device = nl.value, 0, nl.value, device
        self.n_local, self.edges_local, self.stream_bytes_local = nl.value, el.value, sl.value
        self.n_items, self.chunk = ni.value, ch.value
        self.edges = el.value
        return self

    def grid_info(self) -> dict[str, np.ndarray]:
        """cell_of_node, component_id, component_sizes of a device-built graph."""
        r, c, nc = C.c_uint32(), C.c_uint32(), C.c_uint64()
        check(lib().sb_graph_grid_info(self._h, C.byref(r), C.byref(c), None, None, None, C.byref(nc)))
        cell = np.zeros(self.n, np.uint32)
        comp = np.zeros(self.n, np.uint32)
        sizes = np.zeros(max(nc.value, 1), np.uint32)
        check(lib().sb_graph_grid_info(self._h, None, None, ptr(cell), ptr(comp), ptr(sizes), None))
        return dict(rows=r.value, cols=c.value, cell_of_node=cell, component_id=comp,
                    component_sizes=sizes[: nc.value])

    def node_count_of_component(self) -> np.ndarray:
        gi = self.grid_info()
        return gi["component_sizes"][gi["component_id"]]

    def download(self) -> tuple[np.ndarray, np.ndarray, np.ndarray]:
        """(offsets, degrees, stream) of the device CSR slice."""
        off = np.zeros(self.n_local + 1, np.uint64)
        deg = np.zeros(max(self.n_local, 1), np.uint32)
        st = np.zeros(max(self.stream_bytes_local, 1), np.uint8)
        check(lib().sb_graph_download(self._h, ptr(off), ptr(deg), ptr(st)))
        return off, deg[: self.n_local], st[: self.stream_bytes_local]

    def degrees(self) -> np.ndarray:
        """Degrees of the local nodes (device copy)."""
        deg = np.zeros(max(self.n_local, 1), np.uint32)
        check(lib().sb_graph_download(self._h, None, ptr(deg), None))
        return deg[: self.n_local]

    @classmethod
    def from_raw(cls, n, offsets, degrees, stream, device=0, node_range=None):
        """Upload raw arrays (used to exercise the upload-time stream validation)."""
        self = cls.__new__(cls)
        off = np.ascontiguousarray(offsets, np.uint64)
        deg = np.ascontiguousarray(degrees, np.uint32)
        st = np.ascontiguousarray(np.concatenate([np.asarray(stream, np.uint8), np.zeros(64, np.uint8)]))
        v0, v1 = node_range if node_range is not None else (0, n)
        self._h = C.c_void_p()
        check(lib().sb_graph_create(n, ptr(off), ptr(deg), ptr(st), int(off[n]), None, v0, v1, device,
                                    C.byref(self._h)))
        self.n, self.v0, self.v1, self.device = n, v0, v1, device
        self.n_local = v1 - v0
        return self

    def wait(self) -> None:
        """Completes an asynchronous upload (raises RuntimeError on a malformed stream)."""
        check(lib().sb_graph_wait(self._h))

    def local_metrics(self, v0: int = 0, v1: int | None = None) -> dict[str, np.ndarray]:
        """Exact control / controllability / clustering for nodes [v0, v1).

        Needs the full graph on this device (node_range (0, N)); see sb_local_metrics."""
        v1 = self.n if v1 is None else v1
        nl = max(v1 - v0, 0)
        f = [np.zeros(nl, np.float64) for _ in range(3)]
        u = [np.zeros(nl, np.uint64) for _ in range(2)]
        check(lib().sb_local_metrics(self._h, v0, v1, *[ptr(x) for x in f], *[ptr(x) for x in u]))
        return dict(zip(["control", "controllability", "clustering", "edges_among", "n2"], f + u))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sb_graph_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


SCHEDULES = {"auto": 0, "group": SB_HB_SCHEDULE_GROUP, "items": SB_HB_SCHEDULE_WARP}


class HyperBall:
    """HyperBallState on one GPU with iterate_once / run."""

    def __init__(self, graph: CompressedCsr | DeviceGraph, params: HllParams | int,
                 depth_limit: int | None = None, device: int = 0, skip_unchanged: bool = False,
                 node_range: tuple[int, int] | None = None, interval: bool = False, schedule: str = "auto",
                 wavefront: bool = False):
        """schedule: "auto" (16-node shared-gather groups sized to the device, per-node work
        items elsewhere), "group" (groups wherever rows overlap densely, any graph size) or
        "items" (per-warp work items only).  wavefront: run the first run() over an
        asynchronously uploading graph as a wavefront over the upload chunks whatever its
        size (default: streams >= 1 GB).  Every choice gives identical results."""
        self.params = params if isinstance(params, HllParams) else HllParams(params)
        self.graph = graph if isinstance(graph, DeviceGraph) else DeviceGraph(graph, device, node_range)
        self.depth_limit = depth_limit
        self._h = C.c_void_p()
        if schedule not in SCHEDULES:
            raise ValueError(f"schedule must be one of {sorted(SCHEDULES)}")
        flags = ((SB_HB_SKIP_UNCHANGED if skip_unchanged else 0) | (SB_HB_INTERVAL if interval else 0)
                 | SCHEDULES[schedule] | (SB_HB_WAVEFRONT if wavefront else 0))
        check(lib().sb_hb_create(self.graph._h, self.params.p, int(depth_limit or 0), flags, C.byref(self._h)))
        self._comm = None

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().sb_hb_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    # ---- Alg. 1 ------------------------------------------------------------
    def iterate_once(self) -> float:
        """One union/estimate/accumulate pass; returns max_v (c_t - c_{t-1}) (global with a comm)."""
        mx, conv, fin = C.c_double(), C.c_int(), C.c_int()
        check(lib().sb_hb_step(self._h, C.byref(mx), C.byref(conv), C.byref(fin)))
        return mx.value

    def run(self) -> int:
        it, conv = C.c_uint32(), C.c_int()
        check(lib().sb_hb_run(self._h, C.byref(it), C.byref(conv)))
        return it.value

    def step_compute(self) -> float:
        mx = C.c_double()
        check(lib().sb_hb_step_compute(self._h, C.byref(mx)))
        return mx.value

    def step_finish(self, global_max: float) -> tuple[bool, bool]:
        conv, fin = C.c_int(), C.c_int()
        check(lib().sb_hb_step_finish(self._h, float(global_max), C.byref(conv), C.byref(fin)))
        return bool(conv.value), bool(fin.value)

    @staticmethod
    def exchange_local(shards: list["HyperBall"]) -> None:
        arr = (C.c_void_p * len(shards))(*[s._h.value for s in shards])
        check(lib().sb_hb_exchange_local(arr, len(shards)))

    def attach_comm(self, comm: Comm, bounds) -> None:
        b = np.ascontiguousarray(bounds, np.uint64)
        check(lib().sb_hb_attach_comm(self._h, comm._h, ptr(b)))
        self._comm = comm

    def ipc_handles(self) -> bytes:
        """CUDA IPC handles of this rank's planes / changed flags (for attach_peers)."""
        buf = C.create_string_buffer(SB_IPC_HANDLE_BYTES)
        check(lib().sb_hb_ipc_handles(self._h, buf, SB_IPC_HANDLE_BYTES))
        return buf.raw

    def attach_peers(self, rank: int, handles: list[bytes], bounds) -> None:
        """Fused P2P exchange: the union epilogue stores rows into every peer replica."""
        b = np.ascontiguousarray(bounds, np.uint64)
        blob = b"".join(handles)
        assert len(blob) == len(handles) * SB_IPC_HANDLE_BYTES
        check(lib().sb_hb_attach_peers(self._h, len(handles), rank, blob, ptr(b)))

    def reset(self) -> None:
        check(lib().sb_hb_reset(self._h))

    # ---- read-back ---------------------------------------------------------
    def registers(self, which: str = "latest", v0: int = 0, v1: int | None = None) -> np.ndarray:
        """Registers in the reference packed layout (hll.hpp:31-32)."""
        v1 = self.graph.n if v1 is None else v1
        out = np.zeros(max((v1 - v0) * self.params.row_bytes, 1), np.uint8)
        w = SB_REGS_LATEST if which == "latest" else SB_REGS_PREVIOUS
        check(lib().sb_hb_read_registers(self._h, w, v0, v1, ptr(out)))
        return out[: (v1 - v0) * self.params.row_bytes]

    def set_registers(self, packed: np.ndarray) -> None:
        a = np.ascontiguousarray(packed, np.uint8)
        assert a.size == self.graph.n * self.params.row_bytes
        check(lib().sb_hb_set_registers(self._h, ptr(a)))

    def state(self, with_registers: bool = False) -> HyperBallState:
        nl = self.graph.n_local
        c, cp, sd, sd2 = (np.zeros(nl, np.float64) for _ in range(4))
        ch = np.zeros(nl, np.uint8)
        t, conv, fin = C.c_uint32(), C.c_int(), C.c_int()
        check(lib().sb_hb_read_state(self._h, ptr(c), ptr(cp), ptr(sd), ptr(sd2), ptr(ch), C.byref(t),
                                     C.byref(conv), C.byref(fin)))
        regs = self.registers() if with_registers else None
        return HyperBallState(regs, cp, c, sd, sd2, ch, t.value, bool(conv.value), bool(fin.value), self.stats())

    @property
    def t(self) -> int:
        t = C.c_uint32()
        check(lib().sb_hb_read_state(self._h, None, None, None, None, None, C.byref(t), None, None))
        return t.value

    @property
    def finished(self) -> bool:
        fin = C.c_int()
        check(lib().sb_hb_read_state(self._h, None, None, None, None, None, None, None, C.byref(fin)))
        return bool(fin.value)

    def stats(self) -> list[dict]:
        cnt = C.c_uint32()
        check(lib().sb_hb_stats(self._h, None, 0, C.byref(cnt)))
        arr = (sb_iter_stats * max(cnt.value, 1))()
        check(lib().sb_hb_stats(self._h, arr, cnt.value, C.byref(cnt)))
        return [{k: getattr(arr[i], k) for k, _ in sb_iter_stats._fields_} for i in range(cnt.value)]

    def metrics(self, nv: np.ndarray, deg: np.ndarray) -> dict[str, np.ndarray]:
        """MD, IHH, Tekl, PV, first/second moment for the local range."""
        nl = self.graph.n_local
        nv = np.ascontiguousarray(nv, np.uint32)
        deg = np.ascontiguousarray(deg, np.uint32)
        outs = [np.zeros(nl, np.float64) for _ in range(6)]
        check(lib().sb_hb_metrics(self._h, ptr(nv), ptr(deg), *[ptr(o) for o in outs]))
        return dict(zip(["md", "ihh", "tekl", "pv", "m1", "m2"], outs))

    def stream_handle(self) -> int:
        return lib().sb_hb_stream(self._h) or 0


def run(graph: CompressedCsr, params: HllParams | int, depth_limit: int | None = None,
        device: int = 0, skip_unchanged: bool = False) -> HyperBallState:
    """hyperball::run: init, iterate until converged or depth reached."""
    hb = HyperBall(graph, params, depth_limit, device, skip_unchanged)
    hb.run()
    return hb.state(with_registers=True)

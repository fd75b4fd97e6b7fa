"""CompressedCsr: the reference's delta-LEB128 CSR, host side.

Arrays follow SPEC.md:174-177 exactly: ``offsets`` u64[N+1] byte offsets,
``degrees`` u32[N], ``stream`` u8 (per row: first id absolute, then strictly
positive deltas, LEB128 per leb128.hpp:12-39).  Construction, VGACSR03 I/O
(layout :253) and Hilbert renumbering run in the native
library; arrays are zero-copy views of the native object.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import check, lib, ptr, sb_csr_desc


def leb128_encode(value: int) -> bytes:
    """Unsigned LEB128 (leb128.hpp:12-18)."""
    if value < 0:
        raise ValueError("leb128: negative value")
    out = bytearray()
    while value >= 0x80:
        out.append((value & 0x7F) | 0x80)
        value >>= 7
    out.append(value)
    return bytes(out)


def leb128_decode(data: bytes, pos: int = 0) -> tuple[int, int]:
    """Decode one varint at pos -> (value, new_pos); RuntimeError on truncation / >10 bytes (leb128.hpp:28-39)."""
    value = 0
    shift = 0
    for _ in range(10):
        if pos >= len(data):
            raise RuntimeError("leb128: truncated varint")
        b = data[pos]
        pos += 1
        value = (value | ((b & 0x7F) << shift)) & 0xFFFFFFFFFFFFFFFF  # uint64_t, as the reference
        if not b & 0x80:
            return value, pos
        shift += 7
    raise RuntimeError("leb128: varint exceeds 10 bytes")


def encode_neighbor_row(ids) -> bytes:
    """First id absolute, then deltas; strictly increasing input."""
    out = bytearray()
    prev = None
    for w in ids:
        if prev is not None and w <= prev:
            raise ValueError("cgraph: non-increasing neighbour list")
        out += leb128_encode(w if prev is None else w - prev)
        prev = w
    return bytes(out)


def _view(p, n, dtype):
    if n == 0 or not p:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(p, shape=(int(n),)).view(dtype)


def grid_mask(rows: int, cols: int, n_rects: int = 0, rect_min: int = 1, rect_max: int = 1,
              seed: int = 20261017) -> np.ndarray:
    """The (rows, cols) obstacle mask CompressedCsr.synth_grid draws (1 = blocked cell)."""
    m = np.zeros((rows, cols), np.uint8)
    check(lib().sb_grid_synth_mask(rows, cols, n_rects, rect_min, rect_max, seed, ptr(m)))
    return m


class CompressedCsr:
    """Immutable compressed CSR backed by a native sb_csr handle."""

    def __init__(self, handle: int):
        self._h = C.c_void_p(handle)
        d = sb_csr_desc()
        check(lib().sb_csr_describe(self._h, C.byref(d)))
        self.n = int(d.n)
        self.edges = int(d.edges)
        self.stream_len = int(d.stream_len)
        self.offsets = _view(d.offsets, self.n + 1, np.uint64)
        self.degrees = _view(d.degrees, self.n, np.uint32)
        self._stream_padded = _view(d.stream, self.stream_len + 64, np.uint8)
        self.stream = self._stream_padded[: self.stream_len]
        self.component_id = _view(d.component_id, self.n, np.uint32)
        self.component_sizes = _view(d.component_sizes, d.n_components, np.uint32)
        self.cell_of_node = _view(d.cell_of_node, self.n, np.uint32) if d.cell_of_node else None
        self.hilbert_inverse = _view(d.hilbert_inverse, self.n, np.uint32) if d.hilbert_inverse else None
        self.rows, self.cols = int(d.rows), int(d.cols)
        self.origin = (float(d.origin_x), float(d.origin_y))
        self.spacing = float(d.spacing)

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib().sb_csr_destroy(h)
            self._h = None

    # ---- constructors ------------------------------------------------------
    @classmethod
    def synth_grid(cls, rows: int, cols: int, n_rects: int = 0, rect_min: int = 1, rect_max: int = 1,
                   seed: int = 20261017, radius2: int = 0, threads: int = 0) -> "CompressedCsr":
        """Synthetic raster-ordered grid visibility graph (rectangular obstacles, exact integer LOS)."""
        h = C.c_void_p()
        check(lib().sb_csr_synth_grid(rows, cols, n_rects, rect_min, rect_max, seed, radius2, threads,
                                      C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_adjacency(cls, adj) -> "CompressedCsr":
        """adj: list of sorted neighbour lists (build_from_source)."""
        n = len(adj)
        off = np.zeros(n + 1, np.uint64)
        off[1:] = np.cumsum([len(a) for a in adj])
        ids = np.ascontiguousarray(np.concatenate([np.asarray(a, np.uint32) for a in adj])
                                   if n and off[-1] else np.zeros(1, np.uint32), np.uint32)
        h = C.c_void_p()
        check(lib().sb_csr_from_adjacency(n, ptr(off), ptr(ids), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_sorted_csr(cls, adj_offsets, adj_ids) -> "CompressedCsr":
        """Uncompressed sorted CSR arrays (adj_offsets[n+1], adj_ids) -> compressed graph."""
        off = np.ascontiguousarray(adj_offsets, np.uint64)
        ids = np.ascontiguousarray(adj_ids if len(adj_ids) else np.zeros(1), np.uint32)
        h = C.c_void_p()
        check(lib().sb_csr_from_adjacency(off.size - 1, ptr(off), ptr(ids), C.byref(h)))
        return cls(h.value)

    @classmethod
    def from_arrays(cls, offsets, degrees, stream) -> "CompressedCsr":
        """Wrap raw arrays (copied; components recomputed).  No validation beyond offsets[N]."""
        off = np.ascontiguousarray(offsets, np.uint64)
        deg = np.ascontiguousarray(degrees, np.uint32)
        st = np.ascontiguousarray(np.frombuffer(bytes(stream), np.uint8) if not isinstance(stream, np.ndarray)
                                  else stream, np.uint8)
        h = C.c_void_p()
        check(lib().sb_csr_from_arrays(deg.size, ptr(off), ptr(deg), ptr(st) if st.size else None, st.size,
                                       C.byref(h)))
        return cls(h.value)

    @classmethod
    def load_vgacsr(cls, path: str) -> "CompressedCsr":
        h = C.c_void_p()
        check(lib().sb_vgacsr_load(path.encode(), C.byref(h)))
        return cls(h.value)

    # ---- operations --------------------------------------------------------
    def save_vgacsr(self, path: str) -> None:
        check(lib().sb_vgacsr_save(self._h, path.encode()))

    def pin(self, on: bool = True) -> None:
        """Page-lock the stream buffer (pinned H2D for the end-to-end path)."""
        check(lib().sb_csr_pin(self._h, int(on)))

    def hilbert_reorder(self) -> "CompressedCsr":
        h = C.c_void_p()
        check(lib().sb_csr_hilbert_reorder(self._h, C.byref(h)))
        return CompressedCsr(h.value)

    def neighbors(self, v: int) -> np.ndarray:
        """Decoded sorted neighbour ids of v."""
        if not 0 <= v < self.n:
            raise ValueError("node out of range")
        out = np.zeros(max(int(self.degrees[v]), 1), np.uint32)
        check(lib().sb_csr_neighbors(self._h, v, ptr(out)))
        return out[: int(self.degrees[v])]

    def stream_padded(self) -> np.ndarray:
        return self._stream_padded

    def node_count_of_component(self) -> np.ndarray:
        """N_v per node: exact component size."""
        return self.component_sizes[self.component_id]

    def coordinates(self) -> tuple[np.ndarray, np.ndarray]:
        """World (x, y) of each node's cell centre: origin + (col + 0.5, row + 0.5) * spacing."""
        if self.cell_of_node is None or self.cols == 0:
            nan = np.full(self.n, np.nan)
            return nan, nan.copy()
        cell = self.cell_of_node.astype(np.int64)
        row, col = cell // self.cols, cell % self.cols
        return (self.origin[0] + (col + 0.5) * self.spacing, self.origin[1] + (row + 0.5) * self.spacing)

    def partition(self, parts: int) -> np.ndarray:
        """Edge-balanced contiguous node ranges (bounds[parts+1])."""
        b = np.zeros(parts + 1, np.uint64)
        check(lib().sb_partition_edges(self.n, ptr(self.offsets), ptr(self.degrees), parts, ptr(b)))
        return b

    def __repr__(self) -> str:
        return f"CompressedCsr(N={self.n}, |E|={self.edges}, stream={self.stream_len} B)"

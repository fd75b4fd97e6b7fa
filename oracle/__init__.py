"""ctypes wrappers around the parity checker (TEST INFRASTRUCTURE ONLY).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  It is never on the product path.

Two interchangeable back ends expose the same functions:
  * ``port()``      -> oracle/libsboracle.so, the C restatement (sb_oracle.c)
  * ``reference()`` -> oracle/_ref/libsbref.so, the reference's own compiled
                      hll/kernels sources + the SPEC-restated loop (ref_shim.cpp)
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libsboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libsbref.so")

_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class Oracle:
    """One loaded back end; method names follow the reference symbols."""

    def __init__(self, path: str, prefix: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"oracle library missing: {path} (run make -C oracle)")
        self.path = path
        self.kind = "reference" if prefix == "sbref" else "port"
        L = C.CDLL(path)
        self._L = L
        f = lambda name: getattr(L, f"{prefix}_{name}")  # noqa: E731
        self._splitmix = f("splitmix64")
        self._splitmix.restype = C.c_uint64
        self._splitmix.argtypes = [C.c_uint64]
        self._params = f("params")
        self._params.restype = C.c_int
        self._params.argtypes = [C.c_uint, C.POINTER(C.c_uint32), C.POINTER(C.c_double), C.POINTER(C.c_uint32)]
        self._insert = f("insert")
        self._insert.argtypes = [_u8p, C.c_uint64, C.c_uint]
        self._est_sum = f("estimate_from_sum")
        self._est_sum.restype = C.c_double
        self._est_sum.argtypes = [C.c_uint64, C.c_uint32, C.c_uint]
        self._est = f("estimate")
        self._est.restype = C.c_double
        self._est.argtypes = [_u8p, C.c_uint]
        self._enc = f("leb128_encode")
        self._enc.restype = C.c_size_t
        self._enc.argtypes = [C.c_uint64, C.c_char_p]
        self._dec = f("leb128_decode")
        self._dec.restype = C.c_int
        self._dec.argtypes = [C.c_char_p, C.c_size_t, C.POINTER(C.c_size_t), C.POINTER(C.c_uint64)]
        self._init = f("hb_init")
        self._init.restype = C.c_int
        self._init.argtypes = [C.c_uint64, C.c_void_p, C.c_uint, _u8p, _f64p]
        self._iter = f("hb_iterate")
        self._iter.restype = C.c_int
        self._iter.argtypes = [C.c_uint64, _u64p, _u32p, _u8p, C.c_uint64, C.c_uint, C.c_uint32,
                               _u8p, _u8p, _f64p, _f64p, _f64p, _f64p, C.c_uint64, C.c_uint64,
                               C.c_uint, C.POINTER(C.c_double)]
        if self.kind == "port":
            self._nmax = L.sbo_nibble_max
            self._nmax.argtypes = [_u8p, _u8p, C.c_size_t]
            self._harm = L.sbo_harmonic
            self._harm.argtypes = [_u8p, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
            self._metrics = L.sbo_metrics
            self._metrics.argtypes = [C.c_uint64, _f64p, _f64p, _u32p, _u32p] + [_f64p] * 6
            self._local = L.sbo_local_metrics
            self._local.restype = C.c_int
            self._local.argtypes = [C.c_uint64, _u64p, _u32p, _u8p, C.c_uint64, C.c_uint64] + [_f64p] * 3 + [_u64p] * 2
            self._bfs = L.sbo_exact_bfs
            self._bfs.restype = C.c_int
            self._bfs.argtypes = [C.c_uint64, _u64p, _u32p, _u8p, C.c_uint32, _u64p, _u64p, _u32p, _u32p,
                                  C.c_uint32, C.POINTER(C.c_uint32)]
            self._entropy = L.sbo_depth_entropy
            self._entropy.argtypes = [C.c_uint64, _u32p, C.c_uint32, _f64p]
            self._sum_recip = L.sbo_exact_sum_recip
            self._sum_recip.restype = C.c_double
            self._sum_recip.argtypes = [_u32p, C.c_uint64]
        else:
            self._nmax = L.sbref_nibble_max
            self._nmax.argtypes = [_u8p, _u8p, C.c_size_t, C.c_int]
            self._harm = L.sbref_harmonic
            self._harm.argtypes = [_u8p, C.c_size_t, C.c_int, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)]
            self._opsname = L.sbref_ops_name
            self._opsname.restype = C.c_char_p

    # -- primitives -------------------------------------------------------
    def splitmix64(self, x: int) -> int:
        return int(self._splitmix(x))

    def params(self, p: int):
        m, a, rb = C.c_uint32(), C.c_double(), C.c_uint32()
        rc = self._params(p, C.byref(m), C.byref(a), C.byref(rb))
        if rc == 1:
            raise ValueError("hll: precision must be in [4, 16]")
        return m.value, a.value, rb.value

    def insert(self, row: np.ndarray, element: int, p: int) -> None:
        self._insert(row, element, p)

    def nibble_max(self, dst: np.ndarray, src: np.ndarray, scalar: bool = False) -> None:
        if self.kind == "port":
            self._nmax(dst, src, dst.size)
        else:
            self._nmax(dst, src, dst.size, int(scalar))

    def harmonic(self, regs: np.ndarray, scalar: bool = False):
        num, z = C.c_uint64(), C.c_uint32()
        if self.kind == "port":
            self._harm(regs, regs.size, C.byref(num), C.byref(z))
        else:
            self._harm(regs, regs.size, int(scalar), C.byref(num), C.byref(z))
        return num.value, z.value

    def estimate_from_sum(self, num: int, zeros: int, p: int) -> float:
        return float(self._est_sum(num, zeros, p))

    def estimate(self, row: np.ndarray, p: int) -> float:
        return float(self._est(row, p))

    def leb128_encode(self, value: int) -> bytes:
        buf = C.create_string_buffer(16)
        k = self._enc(value, buf)
        return buf.raw[:k]

    def leb128_decode(self, data: bytes, pos: int = 0):
        p = C.c_size_t(pos)
        out = C.c_uint64()
        rc = self._dec(data, len(data), C.byref(p), C.byref(out))
        if rc != 0:
            raise RuntimeError("leb128: malformed varint")
        return out.value, p.value

    # -- HyperBall loop ---------------------------------------------------
    def hb_init(self, n: int, p: int, orig_id: np.ndarray | None = None):
        _, _, rb = self.params(p)
        cur = np.zeros(n * rb, np.uint8)
        c0 = np.zeros(n, np.float64)
        oid = None if orig_id is None else np.ascontiguousarray(orig_id, np.uint32)
        rc = self._init(n, None if oid is None else oid.ctypes.data, p, cur, c0)
        if rc == 1:
            raise ValueError("hyperball: precision out of range or graph empty")
        if rc:
            raise RuntimeError("hyperball init failed")
        return cur, c0

    def hb_iterate(self, csr, p: int, t: int, cur, nxt, c_prev, c_cur, sum_d, sum_d2,
                   v0: int = 0, v1: int | None = None, threads: int = 0) -> float:
        n = csr.n
        v1 = n if v1 is None else v1
        mx = C.c_double()
        rc = self._iter(n, csr.offsets, csr.degrees, csr.stream_padded(), csr.stream_len, p, t,
                        cur, nxt, c_prev, c_cur, sum_d, sum_d2, v0, v1,
                        threads or os.cpu_count() or 1, C.byref(mx))
        if rc == 1:
            raise ValueError("hyperball: invalid argument")
        if rc:
            raise RuntimeError("hyperball: malformed compressed stream")
        return mx.value

    def hb_run(self, csr, p: int, depth_limit: int | None = None, threads: int = 0,
               orig_id: np.ndarray | None = None, per_iteration=None):
        """Alg. 1; per_iteration(t, regs, c) is called after every iterate."""
        n = csr.n
        cur, c_prev = self.hb_init(n, p, orig_id)
        nxt = np.zeros_like(cur)
        c_cur = np.zeros(n, np.float64)
        sum_d = np.zeros(n, np.float64)
        sum_d2 = np.zeros(n, np.float64)
        t = 0
        converged = False
        maxes = []
        while True:
            t += 1
            mx = self.hb_iterate(csr, p, t, cur, nxt, c_prev, c_cur, sum_d, sum_d2, threads=threads)
            maxes.append(mx)
            if per_iteration is not None:
                per_iteration(t, nxt, c_cur)
            if mx <= 0.5:
                converged = True
                break
            if depth_limit and t == depth_limit:
                break
            cur, nxt = nxt, cur
            c_prev, c_cur = c_cur, c_prev
        return dict(registers=nxt, c=c_cur, sum_d=sum_d, sum_d2=sum_d2, iterations=t,
                    converged=converged, max_increase=maxes)

    def metrics(self, sum_d, sum_d2, nv, deg):
        n = sum_d.size
        outs = [np.zeros(n, np.float64) for _ in range(6)]
        if self.kind != "port":
            raise NotImplementedError("metrics are restated in the port only (reference ships none)")
        self._metrics(n, np.ascontiguousarray(sum_d), np.ascontiguousarray(sum_d2),
                      np.ascontiguousarray(nv, np.uint32), np.ascontiguousarray(deg, np.uint32), *outs)
        return dict(zip(["md", "ihh", "tekl", "pv", "m1", "m2"], outs))

    def local_metrics(self, csr, v0: int = 0, v1: int | None = None):
        """Exact control / controllability / clustering, brute force."""
        if self.kind != "port":
            raise NotImplementedError("local metrics are restated in the port only (reference ships none)")
        v1 = csr.n if v1 is None else v1
        nl = v1 - v0
        f = [np.zeros(nl, np.float64) for _ in range(3)]
        u = [np.zeros(nl, np.uint64) for _ in range(2)]
        rc = self._local(csr.n, csr.offsets, csr.degrees, csr.stream_padded(), v0, v1, *f, *u)
        if rc:
            raise RuntimeError("local metrics: malformed graph")
        return dict(zip(["control", "controllability", "clustering", "edges_among", "n2"], f + u))

    def exact_bfs(self, csr, depth_limit: int | None = None, cap: int = 64):
        """Exact per-root BFS: sum_d, sum_d2, reach, depth histogram, entropy."""
        if self.kind != "port":
            raise NotImplementedError("the exact oracle is restated in the port only")
        n = csr.n
        sd, sd2 = np.zeros(n, np.uint64), np.zeros(n, np.uint64)
        reach = np.zeros(n, np.uint32)
        hist = np.zeros(n * cap, np.uint32)
        md = C.c_uint32()
        rc = self._bfs(n, csr.offsets, csr.degrees, csr.stream_padded(), int(depth_limit or 0), sd, sd2, reach,
                       hist, cap, C.byref(md))
        if rc:
            raise RuntimeError("exact bfs: malformed graph")
        if md.value >= cap:
            return self.exact_bfs(csr, depth_limit, cap=2 * md.value + 1)
        ent = np.zeros(n, np.float64)
        self._entropy(n, hist, cap, ent)
        return dict(sum_d=sd, sum_d2=sd2, reach=reach, hist=hist.reshape(n, cap), entropy=ent,
                    max_depth=md.value)

    def exact_sum_recip(self, degs) -> float:
        d = np.ascontiguousarray(degs, np.uint32)
        return float(self._sum_recip(d, d.size))


class SynthCsr:
    """The benchmark grid graph built by the oracle's own generator (sb_synth.c):
    the CSR arrays of SPEC.md:174-177 as zero-copy numpy views of C buffers.
    Duck-types CompressedCsr for Oracle.hb_iterate / hb_run."""

    def __init__(self, rows, cols, n_rects, rect_min, rect_max, seed, radius2, threads=0):
        import weakref
        L = port()._L
        f = L.sbo_synth_grid
        f.restype = C.c_int
        f.argtypes = [C.c_uint32] * 5 + [C.c_uint64, C.c_uint64, C.c_uint] + [C.c_void_p] * 5
        n, off, deg, st, sl = C.c_uint64(), C.c_void_p(), C.c_void_p(), C.c_void_p(), C.c_uint64()
        rc = f(rows, cols, n_rects, rect_min, rect_max, seed, radius2, threads or os.cpu_count() or 1,
               C.byref(n), C.byref(off), C.byref(deg), C.byref(st), C.byref(sl))
        if rc:
            raise RuntimeError(f"sbo_synth_grid failed ({rc})")
        L.sbo_synth_free.argtypes = [C.c_void_p]
        for p in (off, deg, st):
            weakref.finalize(self, L.sbo_synth_free, p.value)
        self.n = n.value
        self.stream_len = sl.value
        view = lambda p, cnt, ct, dt: np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), (cnt,)).view(dt)  # noqa: E731
        self.offsets = view(off, self.n + 1, C.c_uint64, np.uint64)
        self.degrees = view(deg, self.n, C.c_uint32, np.uint32)
        self._stream_padded = view(st, self.stream_len + 256, C.c_uint8, np.uint8)
        self.stream = self._stream_padded[: self.stream_len]
        self.edges = int(self.degrees.sum(dtype=np.uint64))

    def stream_padded(self) -> np.ndarray:
        return self._stream_padded

    def __repr__(self) -> str:
        return f"SynthCsr(N={self.n}, |E|={self.edges}, stream={self.stream_len} B)"


_cache: dict = {}


def port() -> Oracle:
    if "port" not in _cache:
        _cache["port"] = Oracle(PORT_SO, "sbo")
    return _cache["port"]


def reference() -> Oracle:
    if "ref" not in _cache:
        _cache["ref"] = Oracle(REF_SO, "sbref")
    return _cache["ref"]


def reference_available() -> bool:
    return os.path.exists(REF_SO)

"""Generates tests/golden/*.json from the COMPILED REFERENCE primitives.

Run in the build container (needs oracle/_ref/libsbref.so, i.e. the reference
sources under /root/reference/proj/src compiled by oracle/Makefile):

    python tests/golden/make_golden.py

Everything register-level comes from sieveball::splitmix64 / hll_insert /
ops().nibble_max_inplace / ops().harmonic_sum / hll_estimate_from_sum /
leb128_encode (hll.hpp, hll.cpp, kernels*.cpp, leb128.hpp).  The HyperBall
fixtures run the SPEC-restated loop of oracle/ref_shim.cpp over those
primitives on small fixed graphs whose adjacency is stored verbatim.
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def f64hex(x: float) -> str:
    return struct.pack("<d", x).hex()


def leb(v: int) -> bytes:
    out = bytearray()
    while v >= 0x80:
        out.append((v & 0x7F) | 0x80)
        v >>= 7
    out.append(v)
    return bytes(out)


class ArrCsr:
    """Minimal CSR carrier for the oracle (offsets/degrees/stream)."""

    def __init__(self, adj):
        self.n = len(adj)
        rows = []
        for a in adj:
            b = bytearray()
            prev = None
            for w in a:
                b += leb(w if prev is None else w - prev)
                prev = w
            rows.append(bytes(b))
        self.offsets = np.zeros(self.n + 1, np.uint64)
        self.offsets[1:] = np.cumsum([len(r) for r in rows])
        self.degrees = np.array([len(a) for a in adj], np.uint32)
        self.stream = np.frombuffer(b"".join(rows) + b"\0" * 64, np.uint8).copy()
        self.stream_len = int(self.offsets[-1])

    def stream_padded(self):
        return self.stream


def graphs():
    g = {}
    g["P3"] = [[1], [0, 2], [1]]
    g["K2"] = [[1], [0]]
    g["two_triangles"] = [[1, 2], [0, 2], [0, 1], [4, 5], [3, 5], [3, 4]]
    g["star_K1_5"] = [[1, 2, 3, 4, 5], [0], [0], [0], [0], [0]]
    g["isolated_4"] = [[], [], [], []]
    g["path_100"] = [[w for w in (v - 1, v + 1) if 0 <= w < 100] for v in range(100)]
    g["cycle_12"] = [sorted({(v - 1) % 12, (v + 1) % 12}) for v in range(12)]
    rng = np.random.default_rng(20261017)
    n = 300
    m = rng.random((n, n)) < 0.04
    m = np.triu(m, 1)
    m = m | m.T
    g["gnp_300_0.04"] = [np.nonzero(m[v])[0].tolist() for v in range(n)]
    # 20x20 grid, 4-neighbour lattice plus diagonals (diameter 19): long runs
    side = 20
    adj = []
    for r in range(side):
        for c in range(side):
            nb = []
            for dr in (-1, 0, 1):
                for dc in (-1, 0, 1):
                    if (dr or dc) and 0 <= r + dr < side and 0 <= c + dc < side:
                        nb.append((r + dr) * side + c + dc)
            adj.append(sorted(nb))
    g["king_20x20"] = adj
    return g


def main():
    R = oracle.reference()
    out = {"source": "oracle/_ref/libsbref.so (reference hll/kernels sources) ops=" + R._opsname().decode()}
    xs = [0, 1, 2, 3, 42, 1000, 235982, 2**32 - 1, 2**63, 2**64 - 1]
    out["splitmix64"] = {str(x): f"{R.splitmix64(x):016x}" for x in xs}
    out["params"] = {}
    for p in range(4, 17):
        m, a, rb = R.params(p)
        out["params"][str(p)] = {"m": m, "alpha": f64hex(a), "row_bytes": rb}
    ins = {}
    for p in (4, 10, 16):
        rb = (1 << p) // 2
        rows = []
        for e in range(16):
            row = np.zeros(rb, np.uint8)
            R.insert(row, e, p)
            nz = np.nonzero(row)[0]
            j = int(nz[0])
            b = int(row[j])
            idx, rho = (2 * j, b & 0xF) if b & 0xF else (2 * j + 1, b >> 4)
            rows.append([e, idx, rho])
        ins[str(p)] = rows
    out["insert"] = ins
    out["singleton_estimate"] = {}
    for p in range(4, 17):
        row = np.zeros((1 << p) // 2, np.uint8)
        R.insert(row, 1, p)
        out["singleton_estimate"][str(p)] = f64hex(R.estimate(row, p))
    rng = np.random.default_rng(7)
    hs = []
    for p in (4, 5, 6, 8, 10, 12):
        for k in range(4):
            n = (1 << p) // 2
            if k == 0:
                row = np.zeros(n, np.uint8)
            elif k == 1:
                row = np.full(n, 0xFF, np.uint8)
            else:
                row = rng.integers(0, 256, n, dtype=np.uint8)
                if k == 3:  # sparse: few registers set (linear-counting branch)
                    row[rng.random(n) < 0.9] = 0
            num, z = R.harmonic(row)
            hs.append({"p": p, "row": row.tobytes().hex(), "numerator": num, "zeros": z,
                       "estimate": f64hex(R.estimate_from_sum(num, z, p))})
    out["harmonic"] = hs
    nm = []
    for n in (1, 7, 31, 32, 33, 64, 512):
        a = rng.integers(0, 256, n, dtype=np.uint8)
        b = rng.integers(0, 256, n, dtype=np.uint8)
        d = a.copy()
        R.nibble_max(d, b)
        nm.append({"a": a.tobytes().hex(), "b": b.tobytes().hex(), "max": d.tobytes().hex()})
    nm.append({"a": "1f", "b": "f1", "max": "ff"})  # kernels.hpp:22-24
    out["nibble_max"] = nm
    vals = [0, 1, 127, 128, 300, 16383, 16384, 2**21, 2**32 - 1, 2**63, 2**64 - 1]
    out["leb128"] = {str(v): R.leb128_encode(v).hex() for v in vals}

    hb = []
    for name, adj in graphs().items():
        csr = ArrCsr(adj)
        for p in (4, 8, 10, 12):
            for depth in (1, 3, 0):
                hashes = []
                res = R.hb_run(csr, p, depth_limit=depth or None, threads=4,
                               per_iteration=lambda t, regs, c: hashes.append(
                                   hashlib.sha256(regs.tobytes()).hexdigest()))
                hb.append({
                    "graph": name, "p": p, "depth": depth, "iterations": res["iterations"],
                    "converged": res["converged"], "register_sha256_per_iteration": hashes,
                    "sum_d": [f64hex(x) for x in res["sum_d"]] if csr.n <= 100 else
                    hashlib.sha256(res["sum_d"].tobytes()).hexdigest(),
                    "sum_d2_sha256": hashlib.sha256(res["sum_d2"].tobytes()).hexdigest(),
                    "c_sha256": hashlib.sha256(res["c"].tobytes()).hexdigest(),
                    "max_increase": [f64hex(x) for x in res["max_increase"]],
                })
    out["hyperball"] = hb
    out["graphs"] = graphs()
    with open(os.path.join(HERE, "reference_golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print("wrote", os.path.join(HERE, "reference_golden.json"), len(hb), "hyperball cases")


if __name__ == "__main__":
    main()

"""Pins the CPU oracle (test infrastructure) before anything is compared to it.

* SPEC.md known-answer tests (hand-stated in the reference's spec).
* tests/golden/reference_golden.json, produced from the COMPILED reference
  primitives (tests/golden/make_golden.py).
* port (sb_oracle.c) == reference primitives (oracle/_ref) on random inputs,
  when the reference build is present.
"""
import hashlib
import json
import math
import os
import struct

import numpy as np
import pytest

import oracle
from tests.golden.make_golden import ArrCsr

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def f64(h):
    return struct.unpack("<d", bytes.fromhex(h))[0]


BACKENDS = ["port"] + (["reference"] if oracle.reference_available() else [])


@pytest.fixture(params=BACKENDS)
def O(request):
    return oracle.port() if request.param == "port" else oracle.reference()


# ---------------------------------------------------------------- SPEC KATs
def test_spec_leb128_kats(O):
    assert O.leb128_encode(0) == b"\x00"
    assert O.leb128_encode(127) == b"\x7f"
    assert O.leb128_encode(300) == b"\xac\x02"
    assert O.leb128_decode(b"\x00") == (0, 1)
    with pytest.raises(RuntimeError):
        O.leb128_decode(b"\x80")                  # SPEC.md:201 dangling continuation
    with pytest.raises(RuntimeError):
        O.leb128_decode(b"\xff" * 11)             # > 10 bytes (leb128.hpp:38)


def test_spec_leb128_roundtrip(O):
    rng = np.random.default_rng(1)
    for v in rng.integers(0, 2**40, 2000, dtype=np.uint64).tolist():
        enc = O.leb128_encode(int(v))
        assert O.leb128_decode(enc) == (int(v), len(enc))


def test_spec_estimate_kats(O):
    for p in range(4, 17):
        m, _, rb = O.params(p)
        assert O.estimate(np.zeros(rb, np.uint8), p) == 0.0    # SPEC.md:376 all-zero -> 0
    row = np.zeros(512, np.uint8)
    O.insert(row, 12345, 10)
    e = O.estimate(row, 10)
    assert 0.5 <= e <= 2.0
    assert e == pytest.approx(1024 * math.log(1024 / 1023), rel=0, abs=1e-12)


def test_spec_params_invalid(O):
    for p in (0, 3, 17, 64):
        with pytest.raises(ValueError):
            O.params(p)


def test_spec_union_algebra(O):
    rng = np.random.default_rng(3)
    for _ in range(200):
        a, b, c = (rng.integers(0, 256, 64, dtype=np.uint8) for _ in range(3))
        ab = a.copy(); O.nibble_max(ab, b)
        ba = b.copy(); O.nibble_max(ba, a)
        assert np.array_equal(ab, ba)                             # commutative
        aa = a.copy(); O.nibble_max(aa, a)
        assert np.array_equal(aa, a)                              # idempotent
        l = ab.copy(); O.nibble_max(l, c)
        r = b.copy(); O.nibble_max(r, c); O.nibble_max(r, a)
        assert np.array_equal(l, r)                               # associative
        z = a.copy(); O.nibble_max(z, np.zeros_like(a))
        assert np.array_equal(z, a)                               # identity


def test_spec_sketch_of_union(O):
    rng = np.random.default_rng(5)
    for _ in range(100):
        S = set(rng.integers(0, 10**6, 50).tolist())
        T = set(rng.integers(0, 10**6, 50).tolist())
        rs = np.zeros(512, np.uint8)
        rt = np.zeros(512, np.uint8)
        ru = np.zeros(512, np.uint8)
        for e in S:
            O.insert(rs, e, 10)
        for e in T:
            O.insert(rt, e, 10)
        for e in S | T:
            O.insert(ru, e, 10)
        O.nibble_max(rs, rt)
        assert np.array_equal(rs, ru)


def test_spec_convergence_kats():
    P = oracle.port()
    f = P._L.sbo_check_convergence
    f.argtypes = [__import__("ctypes").c_double]
    assert f(0.0) == 1 and f(0.5) == 1 and f(0.51) == 0


# ---------------------------------------------------------------- reference goldens
def test_golden_splitmix64(O):
    for x, h in GOLD["splitmix64"].items():
        assert O.splitmix64(int(x)) == int(h, 16)
    assert O.splitmix64(0) == 0  # hll.hpp:13-20: no increment


def test_golden_params(O):
    for p, d in GOLD["params"].items():
        m, a, rb = O.params(int(p))
        assert (m, rb) == (d["m"], d["row_bytes"]) and a == f64(d["alpha"])


def test_golden_insert(O):
    for p, rows in GOLD["insert"].items():
        p = int(p)
        for e, idx, rho in rows:
            row = np.zeros((1 << p) // 2, np.uint8)
            O.insert(row, e, p)
            b = row[idx >> 1]
            assert ((b >> 4) if idx & 1 else (b & 0xF)) == rho
            assert np.count_nonzero(row) == 1


def test_golden_singleton_estimates(O):
    for p, h in GOLD["singleton_estimate"].items():
        p = int(p)
        row = np.zeros((1 << p) // 2, np.uint8)
        O.insert(row, 1, p)
        assert O.estimate(row, p) == f64(h)


def test_golden_harmonic(O):
    for c in GOLD["harmonic"]:
        row = np.frombuffer(bytes.fromhex(c["row"]), np.uint8).copy()
        assert O.harmonic(row) == (c["numerator"], c["zeros"])
        assert O.estimate_from_sum(c["numerator"], c["zeros"], c["p"]) == f64(c["estimate"])


def test_golden_nibble_max(O):
    for c in GOLD["nibble_max"]:
        a = np.frombuffer(bytes.fromhex(c["a"]), np.uint8).copy()
        b = np.frombuffer(bytes.fromhex(c["b"]), np.uint8).copy()
        O.nibble_max(a, b)
        assert a.tobytes().hex() == c["max"]


def test_golden_leb128(O):
    for v, h in GOLD["leb128"].items():
        assert O.leb128_encode(int(v)).hex() == h


@pytest.mark.parametrize("case", range(len(GOLD["hyperball"])))
def test_golden_hyperball_loop(O, case):
    c = GOLD["hyperball"][case]
    csr = ArrCsr(GOLD["graphs"][c["graph"]])
    hashes = []
    res = O.hb_run(csr, c["p"], depth_limit=c["depth"] or None, threads=2,
                   per_iteration=lambda t, regs, cc: hashes.append(hashlib.sha256(regs.tobytes()).hexdigest()))
    assert res["iterations"] == c["iterations"]
    assert res["converged"] == c["converged"]
    assert hashes == c["register_sha256_per_iteration"]
    assert [f64(x) for x in c["max_increase"]] == res["max_increase"]
    if isinstance(c["sum_d"], list):
        assert [f64(x) for x in c["sum_d"]] == res["sum_d"].tolist()
    else:
        assert hashlib.sha256(res["sum_d"].tobytes()).hexdigest() == c["sum_d"]
    assert hashlib.sha256(res["sum_d2"].tobytes()).hexdigest() == c["sum_d2_sha256"]
    assert hashlib.sha256(res["c"].tobytes()).hexdigest() == c["c_sha256"]


# ---------------------------------------------------------------- SPEC hyperball examples
def test_spec_hyperball_examples():
    P = oracle.port()
    r = P.hb_run(ArrCsr([[]]), 10)                         # isolated node
    assert r["iterations"] == 1 and r["converged"] and r["sum_d"][0] == 0.0
    r = P.hb_run(ArrCsr([[1], [0]]), 12)                   # K2, p=12: MD ~ 1
    assert r["sum_d"] == pytest.approx([1.0, 1.0], rel=0.05)
    adj = [[w for w in (v - 1, v + 1) if 0 <= w < 100] for v in range(100)]
    r = P.hb_run(ArrCsr(adj), 8)                           # 100-node path
    assert 95 <= r["iterations"] <= 101
    star = [[1, 2, 3, 4, 5], [0], [0], [0], [0], [0]]      # K_{1,5}
    cur, c0 = P.hb_init(6, 12)
    nxt = np.zeros_like(cur)
    c1 = np.zeros(6)
    sd, sd2 = np.zeros(6), np.zeros(6)
    P.hb_iterate(ArrCsr(star), 12, 1, cur, nxt, c0, c1, sd, sd2)
    assert c1[0] == pytest.approx(6, rel=0.05) and np.allclose(c1[1:], 2, rtol=0.05)
    assert np.all(c1 >= c0)                                # monotone


def test_spec_metrics_kats():
    P = oracle.port()
    nv = np.array([3, 3, 4, 4, 2, 1], np.uint32)
    sd = np.array([3.0, 2.0, 6.0, 9.0, 1.0, 0.0])          # P3 end, P3 centre, N=4 path-end MD=2, MD=3
    sd2 = np.array([5.0, 2.0, 0, 0, 1.0, 0.0])
    deg = np.array([1, 2, 1, 1, 1, 0], np.uint32)
    m = P.metrics(sd, sd2, nv, deg)
    assert m["md"][0] == 1.5 and m["md"][1] == 1.0
    assert m["ihh"][2] == pytest.approx(1 / 3)
    assert math.isnan(m["ihh"][1])                             # MD=1 -> NaN
    assert m["pv"][2] == 0.0 and m["pv"][1] == 1.0
    assert m["tekl"][1] == 0.0
    assert m["m2"][0] == 2.5 and m["m1"][4] == 1.0
    assert math.isnan(m["md"][5])


def test_metrics_md_below_one():
    """An HLL under-estimate can give MD < 1 (RA < 0): integration_pv stays in
    [0, 1] and integration_hh is NaN (pre MD > 1),
    in the port, the scalar Python forms and the C++ facade's closed forms alike."""
    from paper_2604_08374_b200 import metrics as M
    P = oracle.port()
    nv = np.array([10, 10, 10], np.uint32)
    sd = np.array([8.1, 9.0, 9.9])                              # MD = 0.9, 1.0, 1.1
    m = P.metrics(sd, np.zeros(3), nv, np.ones(3, np.uint32))
    assert m["pv"][0] == 1.0 and m["pv"][1] == 1.0 and 0.0 < m["pv"][2] < 1.0
    assert math.isnan(m["ihh"][0]) and math.isnan(m["ihh"][1]) and m["ihh"][2] > 0
    assert M.integration_pv(0.9, 10) == 1.0 and math.isnan(M.integration_hh(0.9, 10))
    assert M.integration_hh(1.1, 10) == pytest.approx(m["ihh"][2])


@pytest.mark.skipif(not oracle.reference_available(), reason="reference build absent")
def test_port_equals_reference_random():
    P, R = oracle.port(), oracle.reference()
    rng = np.random.default_rng(11)
    for n in (1, 4, 8, 16, 31, 32, 33, 512, 4096):
        a = rng.integers(0, 256, n, dtype=np.uint8)
        b = rng.integers(0, 256, n, dtype=np.uint8)
        x, y = a.copy(), a.copy()
        P.nibble_max(x, b)
        R.nibble_max(y, b)
        assert np.array_equal(x, y)
        assert P.harmonic(a) == R.harmonic(a)
    for p in range(4, 17):
        for _ in range(5):
            row = rng.integers(0, 256, (1 << p) // 2, dtype=np.uint8)
            row[rng.random(row.size) < rng.random()] = 0
            assert P.estimate(row, p) == R.estimate(row, p)

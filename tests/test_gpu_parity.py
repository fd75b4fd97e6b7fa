"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle.

Bar (BASELINE.json north_star): HLL registers bit-exact after EVERY
iteration; c, sum_d, sum_d2, max increase and the iteration count identical
(stronger than the 1e-6 metric tolerance); metrics within 1e-6 relative.
"""
import hashlib
import json
import os
import struct

import numpy as np
import pytest

import oracle
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, HllParams, HyperBall
from tests.golden.make_golden import ArrCsr

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_golden.json")))


def f64(h):
    return struct.unpack("<d", bytes.fromhex(h))[0]


def csr_of(adj):
    return CompressedCsr.from_adjacency(adj)


def lockstep(csr, p, depth, O, skip=False, threads=0, interval=False, schedule="auto"):
    """Run GPU and oracle side by side; assert bit-exact state after every iteration."""
    hb = HyperBall(csr, HllParams(p), depth, skip_unchanged=skip, interval=interval, schedule=schedule)
    n = csr.n
    cur, c_prev = O.hb_init(n, p)
    assert np.array_equal(hb.registers(), cur), "init registers"
    st = hb.state()
    assert np.array_equal(st.c_curr, c_prev), "c_0"
    nxt = np.zeros_like(cur)
    c_cur = np.zeros(n)
    sd, sd2 = np.zeros(n), np.zeros(n)
    t = 0
    while True:
        t += 1
        mg = hb.iterate_once()
        mo = O.hb_iterate(csr, p, t, cur, nxt, c_prev, c_cur, sd, sd2, threads=threads)
        regs = hb.registers()
        if not np.array_equal(regs, nxt):
            bad = np.nonzero(regs != nxt)[0]
            raise AssertionError(f"registers differ at t={t}: {bad.size} bytes, first node {bad[0] // (1 << (p - 1))}")
        s = hb.state()
        assert s.t == t
        assert np.array_equal(s.c_curr, c_cur), f"c_t at t={t}"
        assert np.array_equal(s.c_prev, c_prev), f"c_(t-1) at t={t}"
        assert np.array_equal(s.sum_d, sd), f"sum_d at t={t}"
        assert np.array_equal(s.sum_d2, sd2), f"sum_d2 at t={t}"
        assert mg == mo, f"max increase at t={t}: {mg} vs {mo}"
        conv = mo <= 0.5
        fin = conv or (depth is not None and t == depth)
        assert s.converged == conv and s.finished == fin
        if fin:
            break
        cur, nxt = nxt, cur
        c_prev, c_cur = c_cur, c_prev
    return t


@pytest.fixture(scope="module")
def c1():
    # C1: 64x64 grid, 20 rectangles of 2..9 cells, unlimited radius
    return CompressedCsr.synth_grid(64, 64, 20, 2, 9, 20261017, 0)


# ---------------------------------------------------------------- golden (reference-generated) fixtures
@pytest.mark.parametrize("schedule", ["auto", "group", "items"])
@pytest.mark.parametrize("case", range(len(GOLD["hyperball"])))
def test_gpu_matches_reference_golden(case, schedule):
    c = GOLD["hyperball"][case]
    csr = csr_of(GOLD["graphs"][c["graph"]])
    hb = HyperBall(csr, HllParams(c["p"]), c["depth"] or None, schedule=schedule)
    hashes, maxes = [], []
    while not hb.finished:
        maxes.append(hb.iterate_once())
        hashes.append(hashlib.sha256(hb.registers().tobytes()).hexdigest())
    st = hb.state()
    assert st.t == c["iterations"] and st.converged == c["converged"]
    assert hashes == c["register_sha256_per_iteration"]
    assert maxes == [f64(x) for x in c["max_increase"]]
    if isinstance(c["sum_d"], list):
        assert st.sum_d.tolist() == [f64(x) for x in c["sum_d"]]
    else:
        assert hashlib.sha256(st.sum_d.tobytes()).hexdigest() == c["sum_d"]
    assert hashlib.sha256(st.sum_d2.tobytes()).hexdigest() == c["sum_d2_sha256"]
    assert hashlib.sha256(st.c_curr.tobytes()).hexdigest() == c["c_sha256"]


# ---------------------------------------------------------------- lockstep vs oracle
@pytest.mark.parametrize("schedule", ["auto", "group"])
@pytest.mark.parametrize("p", [4, 5, 6, 7, 8, 9, 10, 11, 12, 13, 14])
def test_gpu_lockstep_c1_depth3(c1, oracle_best, p, schedule):
    assert lockstep(c1, p, 3, oracle_best, schedule=schedule) == 3


@pytest.mark.parametrize("schedule", ["auto", "group", "items"])
@pytest.mark.parametrize("depth", [1, 2, None])
def test_gpu_lockstep_c1_p10(c1, oracle_best, depth, schedule):
    lockstep(c1, 10, depth, oracle_best, schedule=schedule)


@pytest.mark.parametrize("schedule", ["auto", "group"])
@pytest.mark.parametrize("p", [8, 10, 12])
def test_gpu_skip_unchanged_bit_exact(c1, oracle_best, p, schedule):
    lockstep(c1, p, None, oracle_best, skip=True, schedule=schedule)


@pytest.mark.parametrize("p", [15, 16])
def test_gpu_lockstep_large_p(oracle_best, p):
    g = CompressedCsr.synth_grid(24, 24, 6, 2, 5, 3, 0)
    lockstep(g, p, 2, oracle_best)


@pytest.mark.parametrize("schedule", ["auto", "group"])
def test_gpu_lockstep_radius_and_obstacles(oracle_best, schedule):
    g = CompressedCsr.synth_grid(90, 70, 40, 2, 8, 99, 15 * 15)
    lockstep(g, 10, None, oracle_best, schedule=schedule)


@pytest.mark.parametrize("schedule", ["auto", "group", "items"])
def test_gpu_edge_cases(oracle_best, schedule):
    # isolated nodes, empty rows mixed with a clique, a star
    adj = [[], [2, 3, 4], [1, 3, 4], [1, 2, 4], [1, 2, 3], [], [7], [6]]
    for p in (4, 10, 16):
        lockstep(csr_of(adj), p, None, oracle_best, schedule=schedule)
    lockstep(csr_of([[]]), 10, None, oracle_best, schedule=schedule)
    # a dense 300-clique: one group path window holds every id of 8 identical-but-self rows
    clique = [[w for w in range(300) if w != v] for v in range(300)]
    lockstep(csr_of(clique), 10, 2, oracle_best, schedule=schedule)


def test_gpu_schedule_flags_rejected():
    g = csr_of([[1], [0]])
    with pytest.raises(ValueError):
        HyperBall(g, 10, schedule="bogus")


# ---------------------------------------------------------------- interval (sparse-table) variant
@pytest.mark.parametrize("p", [4, 5, 6, 8, 9, 10, 11, 12, 14, 16])
def test_gpu_interval_lockstep_c1(c1, oracle_best, p):
    lockstep(c1, p, None if p <= 12 else 2, oracle_best, interval=True)


@pytest.mark.parametrize("p", [6, 10])
def test_gpu_interval_radius_obstacles(oracle_best, p):
    g = CompressedCsr.synth_grid(90, 70, 40, 2, 8, 99, 15 * 15)
    lockstep(g, p, None, oracle_best, interval=True)
    g = CompressedCsr.synth_grid(60, 80, 0, 1, 1, 5, 20 * 20)  # open grid: long runs
    lockstep(g, p, None, oracle_best, interval=True)


@pytest.mark.parametrize("case", range(len(GOLD["hyperball"])))
def test_gpu_interval_matches_reference_golden(case):
    c = GOLD["hyperball"][case]
    hb = HyperBall(csr_of(GOLD["graphs"][c["graph"]]), HllParams(c["p"]), c["depth"] or None, interval=True)
    hashes = []
    while not hb.finished:
        hb.iterate_once()
        hashes.append(hashlib.sha256(hb.registers().tobytes()).hexdigest())
    assert hashes == c["register_sha256_per_iteration"]
    assert hashlib.sha256(hb.state().sum_d2.tobytes()).hexdigest() == c["sum_d2_sha256"]


def test_gpu_interval_long_runs_peel(oracle_best):
    # a 2600-clique: runs of 2599 ids exceed the 2^(K+1) table span (K capped at 10)
    n = 2600
    adj = [[w for w in range(n) if w != v] for v in range(n)]
    g = csr_of(adj)
    lockstep(g, 10, 2, oracle_best, interval=True)


def test_gpu_interval_rejects_bad_flags():
    g = csr_of([[1], [0]])
    with pytest.raises(ValueError):
        HyperBall(g, 10, interval=True, skip_unchanged=True)


@pytest.mark.parametrize("p", [4, 5, 6, 7, 8, 9, 10, 12])
def test_gpu_interval_random_registers(oracle_best, p):
    g = CompressedCsr.synth_grid(30, 30, 5, 2, 4, p, 0)
    n, rb = g.n, (1 << p) // 2
    rng = np.random.default_rng(100 + p)
    regs = rng.integers(0, 256, n * rb, dtype=np.uint8)
    hb = HyperBall(g, p, None, interval=True)
    hb.set_registers(regs)
    c_prev = hb.state().c_curr.copy()
    nxt = np.zeros_like(regs)
    c_cur, sd, sd2 = np.zeros(n), np.zeros(n), np.zeros(n)
    oracle_best.hb_iterate(g, p, 1, regs, nxt, c_prev, c_cur, sd, sd2)
    hb.iterate_once()
    assert np.array_equal(hb.registers(), nxt)


# ---------------------------------------------------------------- random registers (all nibble values)
@pytest.mark.parametrize("schedule", ["auto", "group"])
@pytest.mark.parametrize("p", list(range(4, 17)))
def test_gpu_random_registers_one_step(oracle_best, p, schedule):
    g = CompressedCsr.synth_grid(20, 20, 4, 2, 4, p, 0)
    n, rb = g.n, (1 << p) // 2
    rng = np.random.default_rng(p)
    regs = rng.integers(0, 256, n * rb, dtype=np.uint8)
    regs[rng.random(regs.size) < 0.3] = 0
    hb = HyperBall(g, p, None, schedule=schedule)
    hb.set_registers(regs)
    assert np.array_equal(hb.registers(), regs), "packed <-> bit-sliced round trip"
    c_prev = np.array([oracle_best.estimate(regs[v * rb:(v + 1) * rb].copy(), p) for v in range(n)])
    assert np.array_equal(hb.state().c_curr, c_prev)
    nxt = np.zeros_like(regs)
    c_cur, sd, sd2 = np.zeros(n), np.zeros(n), np.zeros(n)
    mo = oracle_best.hb_iterate(g, p, 1, regs, nxt, c_prev, c_cur, sd, sd2)
    mg = hb.iterate_once()
    assert np.array_equal(hb.registers(), nxt)
    s = hb.state()
    assert np.array_equal(s.c_curr, c_cur) and np.array_equal(s.sum_d, sd) and mg == mo


# ---------------------------------------------------------------- sharding (same process, one GPU)
@pytest.mark.parametrize("parts", [2, 3, 5])
def test_gpu_local_shards_identical(c1, parts):
    p = 10
    ref = HyperBall(c1, p, None)
    ref.run()
    bounds = c1.partition(parts)
    shards = [HyperBall(c1, p, None, node_range=(int(bounds[i]), int(bounds[i + 1]))) for i in range(parts)]
    while True:
        mx = max(s.step_compute() for s in shards)
        HyperBall.exchange_local(shards)
        fins = [s.step_finish(mx)[1] for s in shards]
        assert len(set(fins)) == 1
        if fins[0]:
            break
    whole = ref.state(with_registers=True)
    for i, s in enumerate(shards):
        st = s.state()
        a, b = int(bounds[i]), int(bounds[i + 1])
        assert st.t == whole.t
        assert np.array_equal(st.sum_d, whole.sum_d[a:b])
        assert np.array_equal(st.c_curr, whole.c_curr[a:b])
        assert np.array_equal(s.registers(), whole.registers)  # full replica everywhere


# ---------------------------------------------------------------- metrics, errors, determinism
def test_gpu_metrics(c1, oracle_port):
    hb = HyperBall(c1, 10, None)
    hb.run()
    s = hb.state()
    nv = c1.node_count_of_component()
    m = hb.metrics(nv, c1.degrees)
    o = oracle_port.metrics(s.sum_d, s.sum_d2, nv, c1.degrees)
    for k in m:
        a, b = m[k], o[k]
        assert np.array_equal(np.isnan(a), np.isnan(b))
        ok = ~np.isnan(a)
        assert np.allclose(a[ok], b[ok], rtol=1e-6, atol=0), k


def test_gpu_errors():
    g = csr_of([[1], [0]])
    with pytest.raises(ValueError):
        HyperBall(g, 3)
    with pytest.raises(ValueError):
        HyperBall(g, 17)
    # truncated varint
    with pytest.raises(RuntimeError):
        DeviceGraph.from_raw(2, [0, 1, 2], [1, 1], [0x81, 0x80])
    # degree mismatch (row has 2 ids, degree says 1)
    with pytest.raises(RuntimeError):
        DeviceGraph.from_raw(3, [0, 2, 3, 4], [1, 1, 1], [1, 1, 0, 1])
    # non-increasing (delta 0)
    with pytest.raises(RuntimeError):
        DeviceGraph.from_raw(3, [0, 2, 3, 4], [2, 1, 1], [1, 0, 0, 1])
    # id out of range
    with pytest.raises(RuntimeError):
        DeviceGraph.from_raw(2, [0, 1, 2], [1, 1], [5, 0])
    # varint longer than 10 bytes (leb128.hpp:38)
    with pytest.raises(RuntimeError):
        DeviceGraph.from_raw(2, [0, 11, 12], [1, 1], [0x81] + [0x80] * 9 + [0x00, 0x00])
    # 6-byte varint whose payload beyond 32 bits is non-zero: id >= N
    with pytest.raises(RuntimeError):
        DeviceGraph.from_raw(2, [0, 6, 7], [1, 1], [0x81, 0x80, 0x80, 0x80, 0x80, 0x01, 0x00])
    hb = HyperBall(g, 10, 1)
    hb.run()
    with pytest.raises(ValueError):
        hb.iterate_once()  # already finished


def test_gpu_determinism_and_reset(c1):
    hb = HyperBall(c1, 10, None)
    hb.run()
    a = hb.state(with_registers=True)
    hb.reset()
    assert hb.t == 0
    hb.run()
    b = hb.state(with_registers=True)
    assert np.array_equal(a.registers, b.registers) and np.array_equal(a.sum_d, b.sum_d)


def test_gpu_pool_reuse_and_release(c1):
    """Freed graph / HyperBall buffers are cached in the stream-ordered pool and reused
    by the next create (same results every cycle); release_cached_memory trims it."""
    from paper_2604_08374_b200 import release_cached_memory
    ref = None
    for cycle in range(4):
        dg = DeviceGraph(c1, async_upload=cycle % 2 == 1)
        hb = HyperBall(dg, HllParams(10), None)
        hb.run()
        sd, regs = hb.state().sum_d, hb.registers()
        del hb, dg
        if ref is None:
            ref = (sd, regs)
        assert np.array_equal(sd, ref[0]) and np.array_equal(regs, ref[1]), cycle
    release_cached_memory(0)
    with pytest.raises(ValueError):
        release_cached_memory(1 << 20)
    hb = HyperBall(c1, 10, None)  # allocations after a trim
    hb.run()
    assert np.array_equal(hb.state().sum_d, ref[0])


def test_gpu_many_handles_pinned_slab_overflow():
    """More live HyperBall handles than the pinned read-back slab has slots (4096):
    the overflow handles fall back to private pinned blocks; every handle still
    steps correctly, and slots are reused after destruction."""
    g = csr_of([[1, 2], [0, 2], [0, 1], []])
    dg = DeviceGraph(g)
    ref = HyperBall(dg, 4, 2)
    ref.run()
    want = ref.state().sum_d
    hs = [HyperBall(dg, 4, 2) for _ in range(4200)]
    for h in hs[::97] + hs[-5:]:
        h.run()
        assert np.array_equal(h.state().sum_d, want)
    del hs[:2000]
    more = [HyperBall(dg, 4, 2) for _ in range(100)]
    for h in more[::9]:
        h.run()
        assert np.array_equal(h.state().sum_d, want)


def test_gpu_hilbert_permutation_equivariance(c1):
    """Hashing original ids makes reordering layout-only."""
    h = c1.hilbert_reorder()
    a = HyperBall(c1, 10, None)
    a.run()
    b = HyperBall(h, 10, None)
    b.run()
    sa, sb_ = a.state(True), b.state(True)
    inv = h.hilbert_inverse.astype(np.int64)
    assert sa.t == sb_.t
    assert np.array_equal(sb_.sum_d, sa.sum_d[inv])
    rb = 512
    ra = sa.registers.reshape(-1, rb)
    rbm = sb_.registers.reshape(-1, rb)
    assert np.array_equal(rbm, ra[inv])


def test_gpu_cpp_facade_tool(oracle_best):
    """tools/sb_hyperball (C++ host over the facade) vs the oracle on C1."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([os.path.join(root, "tools", "sb_hyperball"), "synth", "64", "64", "20", "2", "9",
                        "20261017", "0", "10", "0"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    g = CompressedCsr.synth_grid(64, 64, 20, 2, 9, 20261017, 0)
    ref = oracle_best.hb_run(g, 10)
    nv = g.node_count_of_component().astype(np.float64)
    md = ref["sum_d"] / (nv - 1.0)
    line = [ln for ln in r.stdout.splitlines() if ln.startswith("mean MD")][0]
    assert f"iterations={ref['iterations']}" in r.stdout
    assert float(line.split("=")[1]) == pytest.approx(float(np.mean(md)), rel=1e-6)  # printed with %.6f


def test_gpu_lockstep_c2_full_scale(c2, oracle_best):
    """BASELINE config C2 (212^2 grid, 60 obstacles, radius 44: 42,656 cells, 159 M edges,
    9 iterations) bit-exact after every iteration against the compiled reference
    primitives; C3 is checked against committed reference hashes below."""
    lockstep(c2, 10, None, oracle_best)


# ---------------------------------------------------------------- non-canonical LEB128 (leb128.hpp:28-39)
def noncanonical(csr, rng, frac):
    """Re-encodes csr with a fraction `frac` of its varints padded by zero-payload
    continuation bytes to 6..10 bytes: the same ids, streams the reference decoder
    accepts (it only rejects truncation and > 10 bytes)."""
    from paper_2604_08374_b200.cgraph import leb128_encode
    rows, offs = [], [0]
    for v in range(csr.n):
        out = bytearray()
        prev = None
        for w in csr.neighbors(v):
            b = bytearray(leb128_encode(int(w) if prev is None else int(w) - prev))
            prev = int(w)
            if rng.random() < frac:
                extra = int(rng.integers(6, 11)) - len(b)
                b[-1] |= 0x80
                b += b"\x80" * (extra - 1) + b"\x00"
            out += b
        rows.append(bytes(out))
        offs.append(offs[-1] + len(out))
    return CompressedCsr.from_arrays(np.array(offs, np.uint64), csr.degrees.copy(), b"".join(rows))


@pytest.mark.parametrize("schedule", ["auto", "group"])
@pytest.mark.parametrize("frac", [0.02, 1.0])
def test_gpu_noncanonical_varints_match_reference(c1, oracle_best, frac, schedule):
    """6..10-byte varints decode like the reference (acceptance AND values): registers,
    c and sum_d after every iteration equal the oracle's on the re-encoded stream,
    and the final state equals the canonical stream's.  C1 rows (degree up to ~3,000)
    are cut into 512-id work items, so long varints also sit at item cuts."""
    g = noncanonical(c1, np.random.default_rng(7), frac)
    assert g.stream_len > c1.stream_len
    assert lockstep(g, 10, None, oracle_best, schedule=schedule) >= 3
    a, b = HyperBall(g, 10, None, schedule=schedule), HyperBall(c1, 10, None)
    a.run(), b.run()
    assert np.array_equal(a.registers(), b.registers()) and np.array_equal(a.state().sum_d, b.state().sum_d)
    h = HyperBall(DeviceGraph(g, async_upload=True), 10, None)  # pipelined first pass
    h.run()
    assert np.array_equal(h.registers(), b.registers())
    hi = HyperBall(g, 10, None, interval=True)  # run index from the same stream
    hi.run()
    assert np.array_equal(hi.registers(), b.registers())


def test_gpu_six_byte_varint_accepted_like_reference(oracle_best):
    """`81 80 80 80 80 00` is the 6-byte encoding of 1: the reference converges on
    [[1], [0]] so written; so must the device."""
    raw = CompressedCsr.from_arrays(np.array([0, 6, 7], np.uint64), np.array([1, 1], np.uint32),
                                    bytes([0x81, 0x80, 0x80, 0x80, 0x80, 0x00, 0x00]))
    ref = oracle_best.hb_run(raw, 10)
    hb = HyperBall(raw, 10, None)
    hb.run()
    st = hb.state()
    assert st.t == ref["iterations"] and np.array_equal(hb.registers(), ref["registers"])
    assert np.array_equal(st.sum_d, ref["sum_d"])


# ---------------------------------------------------------------- BASELINE configs at full size
SCALE = os.path.join(os.path.dirname(__file__), "golden", "scale_reference.json")


def _sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def c3():
    from bench import build_graph
    return build_graph("c3", threads=os.cpu_count() or 1)


@pytest.mark.parametrize("mode", ["dense", "skip", "interval", "items"])
def test_gpu_c3_matches_reference_hashes(c3, mode):
    """BASELINE headline config C3 (open 486^2 grid, radius 87: 236,196 cells, 4.79e9
    edges, p=10, full depth): after EVERY iteration the register plane (reference
    packed layout), c_t and the max increase hash-equal the reference CPU path's
    (oracle/_ref, tests/golden/make_scale_golden.py c3); final sum_d / sum_d2 too."""
    gold = json.load(open(SCALE))["c3_p10"]
    gh = gold["graph"]
    assert (c3.n, c3.edges, c3.stream_len) == (gh["nodes"], gh["edges"], gh["stream_bytes"])
    assert _sha(c3.offsets) == gh["offsets_sha256"] and _sha(c3.degrees) == gh["degrees_sha256"]
    assert _sha(c3.stream) == gh["stream_sha256"]
    hb = HyperBall(c3, HllParams(10), None, skip_unchanged=mode == "skip", interval=mode == "interval",
                   schedule="items" if mode == "items" else "auto")
    t = 0
    while not hb.finished:
        mx = hb.iterate_once()
        want = gold["per_iteration"][t]
        t += 1
        assert _sha(hb.registers()) == want["registers_sha256"], f"registers at t={t}"
        assert _sha(hb.state().c_curr) == want["c_sha256"], f"c_t at t={t}"
        assert mx == f64(want["max_increase"]), f"max increase at t={t}"
    st = hb.state()
    assert st.t == gold["iterations"] and st.converged == gold["converged"]
    assert _sha(st.sum_d) == gold["sum_d_sha256"] and _sha(st.sum_d2) == gold["sum_d2_sha256"]


@pytest.mark.parametrize("interval", [False, True], ids=["dense", "interval"])
def test_gpu_c3_pipelined_async_run_matches_reference_hashes(c3, interval):
    """The end-to-end call at C3: sb_graph_create_async + sb_hb_run, whose first
    run is the wavefront over the upload chunks (passes 2.. start while later
    chunks cross PCIe).  Final registers, the previous iteration's registers,
    c_t, sum_d, sum_d2 and every max increase equal the reference CPU path's."""
    gold = json.load(open(SCALE))["c3_p10"]
    hb = HyperBall(DeviceGraph(c3, async_upload=True), HllParams(10), None, interval=interval)
    hb.run()
    st = hb.state()
    assert st.t == gold["iterations"] and st.converged == gold["converged"]
    per = gold["per_iteration"]
    assert _sha(hb.registers()) == per[-1]["registers_sha256"]
    assert _sha(hb.registers("previous")) == per[-2]["registers_sha256"]
    assert _sha(st.c_curr) == per[-1]["c_sha256"]
    assert [x["max_increase"] for x in hb.stats()] == [f64(w["max_increase"]) for w in per]
    assert _sha(st.sum_d) == gold["sum_d_sha256"] and _sha(st.sum_d2) == gold["sum_d2_sha256"]


@pytest.fixture(scope="module")
def c2():
    from bench import build_graph
    g = build_graph("c2", threads=os.cpu_count() or 1)
    assert g.n == 42656
    return g


@pytest.mark.parametrize("p,depth", [(4, None), (6, None), (8, None), (12, None), (14, 2)])
def test_gpu_c4_precision_sweep_lockstep(c2, oracle_best, p, depth):
    """BASELINE C4: the p sweep on the C2 graph, bit-exact after every iteration
    against the reference CPU path (p=10 is test_gpu_lockstep_c2_full_scale)."""
    lockstep(c2, p, depth, oracle_best)

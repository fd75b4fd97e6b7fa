"""sb_graph_create_async: chunked PCIe upload overlapped with the first HyperBall
pass.  Results must be bit-identical to the synchronous upload, and a malformed
stream must still surface as std::runtime_error (RuntimeError) -- at the first
step or at sb_graph_wait instead of at create."""
import numpy as np
import pytest

from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, HyperBall

pytestmark = pytest.mark.gpu


def graphs():
    yield "c1like", CompressedCsr.synth_grid(32, 32, 8, 2, 5, 20261017, 0)  # multi-item nodes
    yield "radius", CompressedCsr.synth_grid(60, 70, 20, 2, 6, 3, 9 * 9)
    yield "tiny", CompressedCsr.from_adjacency([[1], [0, 2], [1], []])


@pytest.mark.parametrize("flags", [{}, {"skip_unchanged": True}, {"interval": True}], ids=["dense", "skip", "interval"])
@pytest.mark.parametrize("p", [6, 10, 12])
@pytest.mark.parametrize("name,g", list(graphs()), ids=[n for n, _ in graphs()])
def test_async_upload_bit_identical(name, g, p, flags):
    ref = HyperBall(g, p, None, **flags)
    ref.run()
    hb = HyperBall(DeviceGraph(g, async_upload=True), p, None, **flags)
    hb.run()
    assert np.array_equal(hb.registers(), ref.registers())
    a, b = hb.state(), ref.state()
    assert a.t == b.t and np.array_equal(a.sum_d, b.sum_d) and np.array_equal(a.sum_d2, b.sum_d2)


def test_async_upload_shards_and_other_users():
    g = CompressedCsr.synth_grid(60, 70, 20, 2, 6, 3, 9 * 9)
    ref = HyperBall(g, 10, None)
    ref.run()
    n = g.n
    parts = [(0, n // 3), (n // 3, n)]
    hs = [HyperBall(DeviceGraph(g, node_range=r, async_upload=True), 10, None, node_range=r) for r in parts]
    while True:
        mx = max(h.step_compute() for h in hs)
        HyperBall.exchange_local(hs)
        if hs[0].step_finish(mx)[1] | hs[1].step_finish(mx)[1]:
            break
    assert np.array_equal(np.concatenate([h.state().sum_d for h in hs]), ref.state().sum_d)
    dg = DeviceGraph(g, async_upload=True)  # local metrics / download wait for the upload themselves
    off, deg, st = dg.download()
    assert np.array_equal(st, g.stream) and np.array_equal(deg, g.degrees)
    assert np.array_equal(DeviceGraph(g, async_upload=True).local_metrics()["clustering"],
                          DeviceGraph(g).local_metrics()["clustering"], equal_nan=True)


def _raw(n, offsets, degrees, stream):
    return CompressedCsr.from_arrays(offsets, degrees, bytes(stream))


def _cut_row(n, deg, bad_at, kind):
    """Node 0 -> ids 1..deg (cut into 512-id work items), malformed at neighbour
    `bad_at`: a zero delta, or a delta that jumps far past N; other rows empty."""
    from paper_2604_08374_b200.cgraph import leb128_encode
    row = bytearray(leb128_encode(1))
    for k in range(1, deg):
        d = 1
        if k == bad_at:
            d = 0 if kind == "zero" else (1 << 31)
        row += leb128_encode(d)
    offs = [0, len(row)] + [len(row)] * (n - 1)
    return n, offs, [deg] + [0] * (n - 1), list(row)


@pytest.mark.parametrize("bad", [
    (2, [0, 1, 2], [1, 1], [0x81, 0x80]),                  # truncated varint
    (3, [0, 2, 3, 4], [1, 1, 1], [1, 1, 0, 1]),             # degree mismatch
    (2, [0, 1, 2], [1, 1], [5, 0]),                         # id out of range
    (2, [0, 5, 6], [1, 1], [0x80, 0x80, 0x80, 0x80, 0x08, 0]),  # id 2^31: far outside the plane
    _cut_row(1600, 1500, 1000, "zero"),                     # zero delta inside the row's 2nd work item
    _cut_row(1600, 1500, 700, "huge"),                      # id jump of 2^31 inside a cut row
], ids=["truncated", "degree", "range", "range_huge", "cut_zero", "cut_huge"])
def test_async_upload_reports_malformed_stream(bad):
    """A malformed row surfaces as RuntimeError (sticky), and the pipelined first
    pass never dereferences its ids: the union CTAs stop once validation has
    flagged the chunk, so the CUDA context stays healthy (the next graph runs)."""
    g = _raw(*bad)
    dg = DeviceGraph(g, async_upload=True)
    hb = HyperBall(dg, 10, None)
    with pytest.raises(RuntimeError):
        hb.iterate_once()
    with pytest.raises(RuntimeError):  # sticky
        hb.iterate_once()
    with pytest.raises(RuntimeError):
        DeviceGraph(g, async_upload=True).wait()
    ok = CompressedCsr.from_adjacency([[1], [0, 2], [1], []])
    h = HyperBall(DeviceGraph(ok, async_upload=True), 10, None)
    h.run()
    ref = HyperBall(ok, 10, None)
    ref.run()
    assert np.array_equal(h.registers(), ref.registers())


@pytest.mark.parametrize("bad", [_cut_row(1600, 1500, 1000, "zero"), _cut_row(1600, 1500, 700, "huge")],
                         ids=["cut_zero", "cut_huge"])
def test_async_upload_interval_malformed_stream(bad):
    """Interval mode counts the run index per upload chunk while the copies are
    still in flight; a malformed chunk stops the count kernels (they never follow
    its item offsets) and surfaces as RuntimeError at create."""
    g = _raw(*bad)
    with pytest.raises(RuntimeError):
        HyperBall(DeviceGraph(g, async_upload=True), 10, None, interval=True)
    ok = CompressedCsr.synth_grid(40, 40, 6, 2, 5, 11, 0)
    h = HyperBall(DeviceGraph(ok, async_upload=True), 10, None, interval=True)
    h.run()
    ref = HyperBall(ok, 10, None)
    ref.run()
    assert np.array_equal(h.registers(), ref.registers())


# ---------------------------------------------------------------- wavefront first run
# sb_hb_run over a graph still uploading runs passes 2, 3, ... on the first
# chunks while later chunks cross PCIe (pipelined_run, sb_hb_api.cu).  Graphs
# whose rows reference only nearby ids (grids with a radius) engage it; the
# result must equal the stepped run on the synchronously uploaded graph in
# every observable: registers (latest and previous), c, sum_d, sum_d2, t,
# convergence, the per-iteration max increases and changed counts.
def wave_graphs():
    yield "grid_r6", CompressedCsr.synth_grid(150, 150, 30, 2, 6, 5, 6 * 6)       # deps +-1-2 chunks
    yield "strip_r3", CompressedCsr.synth_grid(400, 40, 10, 1, 4, 9, 3 * 3)        # long diameter: many passes
    yield "open_r12", CompressedCsr.synth_grid(120, 120, 0, 1, 1, 1, 12 * 12)      # denser rows, group path at p>=9
    yield "global", CompressedCsr.synth_grid(40, 40, 6, 2, 4, 3, 0)                # unlimited radius: every chunk depends on all


def _same_run(a, b):
    assert np.array_equal(a.registers(), b.registers())
    assert np.array_equal(a.registers("previous"), b.registers("previous"))
    sa, sb = a.state(), b.state()
    assert (sa.t, sa.converged, sa.finished) == (sb.t, sb.converged, sb.finished)
    assert np.array_equal(sa.c_curr, sb.c_curr) and np.array_equal(sa.c_prev, sb.c_prev)
    assert np.array_equal(sa.sum_d, sb.sum_d) and np.array_equal(sa.sum_d2, sb.sum_d2)
    ka, kb = a.stats(), b.stats()
    assert [x["max_increase"] for x in ka] == [x["max_increase"] for x in kb]
    assert [x["changed_nodes"] for x in ka] == [x["changed_nodes"] for x in kb]


@pytest.mark.parametrize("interval", [False, True], ids=["dense", "interval"])
@pytest.mark.parametrize("depth", [None, 2, 3, 5])
@pytest.mark.parametrize("p", [4, 6, 10, 12])
@pytest.mark.parametrize("name,g", list(wave_graphs()), ids=[n for n, _ in wave_graphs()])
def test_pipelined_first_run_bit_identical(name, g, p, depth, interval):
    """interval: the wavefront also builds the run index chunk by chunk and a
    sparse table per pass and chunk."""
    ref = HyperBall(g, p, depth)
    ref.run()
    hb = HyperBall(DeviceGraph(g, async_upload=True), p, depth, wavefront=True, interval=interval)
    hb.run()
    _same_run(hb, ref)
    # the handle keeps working: reset and a second (device-resident) run
    hb.reset()
    hb.run()
    _same_run(hb, ref)


def test_pipelined_first_run_converges_inside_the_wavefront():
    """Many small cliques of consecutive ids: every chunk reads only itself, so the
    wavefront starts passes 2..12 while the upload is in flight, but the run
    converges at pass 2.  The speculative passes must leave no trace."""
    k, c = 2000, 8
    adj = [[b * c + j for j in range(c) if j != i] for b in range(k) for i in range(c)]
    g = CompressedCsr.from_adjacency(adj)
    for p in (4, 10):
        ref = HyperBall(g, p, None)
        ref.run()
        for interval in (False, True):
            hb = HyperBall(DeviceGraph(g, async_upload=True), p, None, wavefront=True, interval=interval)
            hb.run()
            assert ref.state().t <= 3
            _same_run(hb, ref)


def _run_storage_overflow_graph():
    """Single-run rows first, then rows of every other id: the run storage sized
    from the first chunks' runs per byte is far too small for the rest."""
    n, w = 6000, 200
    adj = []
    for v in range(n):
        if v < 1000:
            lo = min(max(v - w // 2, 0), n - w - 1)
            adj.append([u for u in range(lo, lo + w + 1) if u != v])
        else:
            lo = min(max(v - w, 0), n - 2 * w - 1)
            adj.append([u for u in range(lo, lo + 2 * w, 2) if u != v])
    return CompressedCsr.from_adjacency(adj)


@pytest.mark.parametrize("p", [6, 10])
def test_pipelined_interval_run_storage_overflow(p):
    """The wavefront's interval passes read a run index filled chunk by chunk
    into storage sized from the first chunks' runs per byte; here the later
    chunks need ~60x more, so the storage grows while passes already run on
    the old one -- same result as the stepped run, also after a reset."""
    g = _run_storage_overflow_graph()
    ref = HyperBall(g, p, None)
    ref.run()
    hb = HyperBall(DeviceGraph(g, async_upload=True), p, None, wavefront=True, interval=True)
    hb.run()
    _same_run(hb, ref)
    hb.reset()
    hb.run()
    _same_run(hb, ref)


def test_async_run_index_growth_for_exact_and_local_metrics():
    """The same uneven graph through the other users of the run index built
    under an asynchronous upload (storage grown per chunk, no wavefront):
    exact local metrics and the interval exact BFS equal the synchronous graph's."""
    from paper_2604_08374_b200 import ExactBfs
    g = _run_storage_overflow_graph()
    ref_lm = DeviceGraph(g).local_metrics()
    lm = DeviceGraph(g, async_upload=True).local_metrics()
    for key in ref_lm:
        assert np.array_equal(lm[key], ref_lm[key], equal_nan=lm[key].dtype.kind == "f"), key
    ref = ExactBfs(DeviceGraph(g), 3)
    ref.run()
    x = ExactBfs(DeviceGraph(g, async_upload=True), 3, interval=True)
    x.run()
    ra, rb = x.result(), ref.result()
    for key in ("sum_d", "sum_d2", "reach"):
        assert np.array_equal(ra[key], rb[key]), key


def test_pipelined_interval_fuzz_case_43x30():
    """The randomised campaign's case (seed 7) whose wavefront read past the
    estimated run storage (before it could grow)."""
    g = CompressedCsr.synth_grid(43, 30, 34, 3, 7, 1218590505, 186)
    for depth in (5, None):
        ref = HyperBall(g, 10, depth)
        ref.run()
        for interval in (True, False):
            hb = HyperBall(DeviceGraph(g, async_upload=True), 10, depth, wavefront=True, interval=interval)
            hb.run()
            _same_run(hb, ref)


@pytest.mark.parametrize("sched", ["group", "items"])
def test_pipelined_first_run_schedules(sched):
    g = CompressedCsr.synth_grid(150, 150, 30, 2, 6, 5, 6 * 6)
    ref = HyperBall(g, 10, None)
    ref.run()
    hb = HyperBall(DeviceGraph(g, async_upload=True), 10, None, schedule=sched, wavefront=True)
    hb.run()
    _same_run(hb, ref)


def _corrupt_middle_row(kind):
    """A valid radius grid (16 upload chunks) with one bad varint in a row of the
    9th chunk: a zero delta, or a delta of 2^31 (ids far outside the plane)."""
    g = CompressedCsr.synth_grid(150, 150, 30, 2, 6, 5, 6 * 6)
    offs, deg, st = g.offsets.copy(), g.degrees.copy(), bytearray(g.stream.tobytes())
    v = g.n * 9 // 16
    a, b = int(offs[v]), int(offs[v + 1])
    row = st[a:b]
    k = len(row) // 2
    while row[k] & 0x80 or row[k - 1] & 0x80:  # a one-byte varint in the middle
        k += 1
    if kind == "zero":
        st[a + k] = 0
        return CompressedCsr.from_arrays(offs, deg, bytes(st))
    new = bytes(st[:a + k]) + bytes([0x80, 0x80, 0x80, 0x80, 0x08]) + bytes(st[a + k + 1:])
    offs[v + 1:] += 4
    return CompressedCsr.from_arrays(offs, deg, new)


@pytest.mark.parametrize("interval", [False, True], ids=["dense", "interval"])
@pytest.mark.parametrize("kind", ["zero", "huge"])
def test_pipelined_first_run_reports_malformed_stream(kind, interval):
    g = _corrupt_middle_row(kind)
    hb = HyperBall(DeviceGraph(g, async_upload=True), 10, None, wavefront=True, interval=interval)
    with pytest.raises(RuntimeError):
        hb.run()
    ok = CompressedCsr.synth_grid(60, 70, 20, 2, 6, 3, 9 * 9)
    h = HyperBall(DeviceGraph(ok, async_upload=True), 10, None)
    h.run()
    ref = HyperBall(ok, 10, None)
    ref.run()
    assert np.array_equal(h.registers(), ref.registers())

"""Host CompressedCsr: LEB128 rows, builder, generator,
components, VGACSR03 persistence, Hilbert reorder, partitions.  CPU only."""
import os
import zlib

import numpy as np
import pytest

import oracle
from paper_2604_08374_b200 import CompressedCsr, encode_neighbor_row, leb128_decode, leb128_encode


def test_leb128_spec_examples():
    assert leb128_encode(0) == b"\x00" and leb128_encode(127) == b"\x7f" and leb128_encode(300) == b"\xac\x02"
    assert leb128_decode(b"\x00") == (0, 1)
    with pytest.raises(RuntimeError):
        leb128_decode(b"\x80")
    with pytest.raises(RuntimeError):
        leb128_decode(b"\xff" * 11)
    rng = np.random.default_rng(0)
    O = oracle.port()
    for v in rng.integers(0, 2**40, 5000).tolist():
        e = leb128_encode(v)
        assert e == O.leb128_encode(v) and leb128_decode(e) == (v, len(e))


def test_row_encoding_spec_example():
    # [100,101,103,1300] -> enc(100) ++ enc(1) ++ enc(2) ++ enc(1197)
    assert encode_neighbor_row([100, 101, 103, 1300]) == b"\x64\x01\x02" + leb128_encode(1197)
    assert encode_neighbor_row([]) == b""
    with pytest.raises(ValueError):
        encode_neighbor_row([3, 3])


def test_builder_spec_examples():
    g = CompressedCsr.from_adjacency([[1], [0, 2], [1]])          # P3
    assert g.degrees.tolist() == [1, 2, 1] and g.component_sizes.tolist() == [3]
    assert [g.neighbors(v).tolist() for v in range(3)] == [[1], [0, 2], [1]]
    t = CompressedCsr.from_adjacency([[1, 2], [0, 2], [0, 1], [4, 5], [3, 5], [3, 4]])
    assert t.component_sizes.tolist() == [3, 3] and t.component_id.tolist() == [0, 0, 0, 1, 1, 1]
    rng = np.random.default_rng(500)                                # G(500, 0.05) round trip
    m = np.triu(rng.random((500, 500)) < 0.05, 1)
    m = m | m.T
    adj = [np.nonzero(m[v])[0].tolist() for v in range(500)]
    g = CompressedCsr.from_adjacency(adj)
    assert all(g.neighbors(v).tolist() == adj[v] for v in range(500))
    assert int(g.offsets[-1]) == g.stream_len and g.edges == int(m.sum())
    with pytest.raises(ValueError):
        CompressedCsr.from_adjacency([[1, 1], [0]])
    with pytest.raises(ValueError):
        CompressedCsr.from_adjacency([[5], [0]])


def test_empty_rows_take_zero_bytes():
    g = CompressedCsr.from_adjacency([[], [2], [1], []])
    assert g.offsets.tolist() == [0, 0, 1, 2, 2]
    assert g.component_sizes.tolist() == [1, 2, 1]


def brute_visible(blocked, r1, c1, r2, c2):
    """Independent LOS: sample the open segment densely in exact rationals and
    test cell interiors (fractions avoid float ties)."""
    from fractions import Fraction as Fr
    x1, y1, x2, y2 = 2 * c1 + 1, 2 * r1 + 1, 2 * c2 + 1, 2 * r2 + 1
    # candidate cells are those whose interior the segment crosses: check the
    # midpoints between consecutive boundary crossings.
    ts = {Fr(0), Fr(1)}
    dx, dy = x2 - x1, y2 - y1
    for X in range(min(x1, x2), max(x1, x2) + 1):
        if X % 2 == 0 and dx:
            ts.add(Fr(X - x1, dx))
    for Y in range(min(y1, y2), max(y1, y2) + 1):
        if Y % 2 == 0 and dy:
            ts.add(Fr(Y - y1, dy))
    ts = sorted(t for t in ts if 0 <= t <= 1)
    for a, b in zip(ts, ts[1:]):
        t = (a + b) / 2
        x, y = x1 + dx * t, y1 + dy * t
        c, r = int(x // 2), int(y // 2)
        if blocked[r][c]:
            return False
    return True


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_generator_matches_brute_force_los(seed):
    rows, cols = 11, 13
    g = CompressedCsr.synth_grid(rows, cols, 6, 1, 4, seed, 0)
    cells = g.cell_of_node
    free = set(cells.tolist())
    blocked = [[(r * cols + c) not in free for c in range(cols)] for r in range(rows)]
    node_of = {int(c): i for i, c in enumerate(cells)}
    for v in range(g.n):
        r1, c1 = divmod(int(cells[v]), cols)
        want = []
        for cell in sorted(free):
            if cell == cells[v]:
                continue
            r2, c2 = divmod(cell, cols)
            if brute_visible(blocked, r1, c1, r2, c2):
                want.append(node_of[cell])
        assert g.neighbors(v).tolist() == want, v


def test_generator_symmetry_radius_and_components():
    g = CompressedCsr.synth_grid(40, 33, 25, 2, 7, 11, 9 * 9)
    adj = [set(g.neighbors(v).tolist()) for v in range(g.n)]
    assert all(v in adj[w] for v in range(g.n) for w in adj[v])     # undirected
    cols = 33
    for v in range(0, g.n, 37):
        r1, c1 = divmod(int(g.cell_of_node[v]), cols)
        for w in adj[v]:
            r2, c2 = divmod(int(g.cell_of_node[w]), cols)
            assert (r1 - r2) ** 2 + (c1 - c2) ** 2 <= 81
    # components == BFS flood fill over the visibility graph
    comp = -np.ones(g.n, np.int64)
    cid = 0
    for s in range(g.n):
        if comp[s] >= 0:
            continue
        comp[s] = cid
        st = [s]
        while st:
            x = st.pop()
            for y in adj[x]:
                if comp[y] < 0:
                    comp[y] = cid
                    st.append(y)
        cid += 1
    assert cid == len(g.component_sizes)
    assert np.array_equal(comp, g.component_id.astype(np.int64))   # ids by first occurrence


def test_open_grid_compression_ratio():
    g = CompressedCsr.synth_grid(60, 60, 0, 1, 1, 0, 22 * 22)      # SPEC.md:703 (AC 6)
    assert g.edges * 4 / g.stream_len >= 3.0


def test_vgacsr_roundtrip_and_errors(tmp_path):
    g = CompressedCsr.synth_grid(30, 30, 10, 2, 5, 4, 0)
    p = str(tmp_path / "g.vgacsr")
    g.save_vgacsr(p)
    h = CompressedCsr.load_vgacsr(p)
    for a in ("offsets", "degrees", "stream", "component_id", "component_sizes", "cell_of_node"):
        assert np.array_equal(getattr(g, a), getattr(h, a)), a
    assert (h.rows, h.cols, h.n, h.edges) == (g.rows, g.cols, g.n, g.edges)
    raw = open(p, "rb").read()
    assert raw[:8] == b"VGACSR03"
    assert int.from_bytes(raw[-4:], "little") == zlib.crc32(raw[:-4])   # trailing CRC32
    bad = tmp_path / "bad"
    bad.write_bytes(b"VGACSR02" + raw[8:])
    with pytest.raises(RuntimeError, match="version"):
        CompressedCsr.load_vgacsr(str(bad))
    bad.write_bytes(b"XXXXXXXX" + raw[8:])
    with pytest.raises(RuntimeError, match="magic"):
        CompressedCsr.load_vgacsr(str(bad))
    flip = bytearray(raw)
    flip[len(raw) // 2] ^= 0x40
    bad.write_bytes(bytes(flip))
    with pytest.raises(RuntimeError, match="checksum"):
        CompressedCsr.load_vgacsr(str(bad))
    bad.write_bytes(raw[: len(raw) // 3])
    with pytest.raises(RuntimeError, match="truncated"):
        CompressedCsr.load_vgacsr(str(bad))

    def with_crc(body: bytes) -> bytes:
        return body + zlib.crc32(body).to_bytes(4, "little")

    # a corrupt header claiming 2^32-1 nodes is rejected before any allocation
    huge = bytearray(raw)
    huge[12:20] = (0xFFFFFFFF).to_bytes(8, "little")
    bad.write_bytes(bytes(huge))
    with pytest.raises(RuntimeError, match="truncated"):
        CompressedCsr.load_vgacsr(str(bad))
    # component ids are checked against C and the sizes against the ids (CRC kept valid)
    n = g.n
    comp_at = len(raw) - 4 - 4 * g.component_sizes.size - 4 * n
    body = bytearray(raw[:-4])
    body[comp_at:comp_at + 4] = (g.component_sizes.size + 7).to_bytes(4, "little")
    bad.write_bytes(with_crc(bytes(body)))
    with pytest.raises(RuntimeError, match="component id"):
        CompressedCsr.load_vgacsr(str(bad))
    body = bytearray(raw[:-4])
    sz_at = len(raw) - 4 - 4 * g.component_sizes.size
    body[sz_at:sz_at + 4] = (int(g.component_sizes[0]) + 1).to_bytes(4, "little")
    bad.write_bytes(with_crc(bytes(body)))
    with pytest.raises(RuntimeError, match="component sizes"):
        CompressedCsr.load_vgacsr(str(bad))


def test_hilbert_reorder_is_a_relabelling(tmp_path):
    g = CompressedCsr.synth_grid(20, 24, 8, 1, 4, 9, 0)
    h = g.hilbert_reorder()
    inv = h.hilbert_inverse
    assert sorted(inv.tolist()) == list(range(g.n))
    fwd = np.empty(g.n, np.int64)
    fwd[inv] = np.arange(g.n)
    for i in range(h.n):
        assert sorted(fwd[g.neighbors(int(inv[i]))].tolist()) == h.neighbors(i).tolist()
    assert abs(h.stream_len - g.stream_len) / g.stream_len < 0.5
    p = str(tmp_path / "h.vgacsr")
    h.save_vgacsr(p)
    assert np.array_equal(CompressedCsr.load_vgacsr(p).hilbert_inverse, inv)


def test_hilbert_order1_convention():
    # order-1 on a 2x2 grid, pairs are (row, col) (SPEC.md:238
    # "Hilbert index of (row, col)"): (0,0)->0, (1,0)->1, (1,1)->2, (0,1)->3
    g = CompressedCsr.synth_grid(2, 2, 0, 1, 1, 0, 0)
    h = g.hilbert_reorder()
    cells = [(int(c) // 2, int(c) % 2) for c in h.cell_of_node]
    assert cells == [(0, 0), (1, 0), (1, 1), (0, 1)]


@pytest.mark.parametrize("parts", [1, 2, 3, 8])
def test_partition_edge_balanced(parts):
    g = CompressedCsr.synth_grid(50, 50, 12, 2, 6, 5, 12 * 12)
    b = g.partition(parts)
    assert b[0] == 0 and b[-1] == g.n and np.all(np.diff(b.astype(np.int64)) >= 0)
    w = g.degrees.astype(np.int64) + 1
    loads = [int(w[int(b[i]):int(b[i + 1])].sum()) for i in range(parts)]
    assert max(loads) - min(loads) <= 2 * int(w.max())


def test_hilbert_components_match_union_find():
    """The reorder permutes components (first-occurrence ids in the new order) instead of
    re-running UnionFind over every edge; both must agree."""
    for args in ((40, 44, 30, 1, 6, 3, 0), (50, 50, 120, 1, 3, 9, 7 * 7)):
        h = CompressedCsr.synth_grid(*args).hilbert_reorder()
        uf = CompressedCsr.from_arrays(h.offsets, h.degrees, h.stream)
        assert np.array_equal(h.component_id, uf.component_id)
        assert np.array_equal(h.component_sizes, uf.component_sizes)

"""Exact local metrics: connectivity, control, controllability, clustering.

CPU: the oracle against the SPEC's worked examples (triangle, star K_{1,5}),
an adjacency-matrix brute force on random G(30, 0.3) and exact
rational arithmetic for the control sum.  GPU: sb_local_metrics bit-equal to
the oracle (acceptance criterion 9) on the same graphs, on
synthetic visibility grids, node sub-ranges and the global-scratch path.
"""
import os
import subprocess
import sys
from fractions import Fraction

import numpy as np
import pytest

import oracle
from paper_2604_08374_b200 import CompressedCsr, DeviceGraph

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def random_graph(n, p, seed):
    rng = np.random.default_rng(seed)
    A = np.triu(rng.random((n, n)) < p, 1)
    A = A | A.T
    adj = [list(np.nonzero(A[v])[0]) for v in range(n)]
    return A, CompressedCsr.from_adjacency(adj)


def brute(A):
    """Adjacency-matrix oracle: control (exact rational), clustering, controllability."""
    n = A.shape[0]
    Ai = A.astype(np.int64)
    deg = Ai.sum(1)
    among = np.diag(Ai @ Ai @ Ai)
    two = ((Ai + Ai @ Ai) > 0)
    np.fill_diagonal(two, False)
    n2 = two.sum(1)
    control = [float(sum((Fraction(1.0 / deg[w]) for w in np.nonzero(A[v])[0]), Fraction(0))) for v in range(n)]
    clus = np.array([among[v] / (float(deg[v]) * float(deg[v] - 1)) if deg[v] >= 2 else np.nan for v in range(n)])
    ctrl = np.array([deg[v] / n2[v] if n2[v] else np.nan for v in range(n)])
    return dict(control=np.array(control), clustering=clus, controllability=ctrl,
                edges_among=among.astype(np.uint64), n2=n2.astype(np.uint64))


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and np.array_equal(a, b, equal_nan=a.dtype.kind == "f")


# ------------------------------------------------------------------ CPU (oracle)
def test_exact_reciprocal_sum_is_correctly_rounded(oracle_port):
    rng = np.random.default_rng(7)
    for _ in range(300):
        hi = 2**32 if rng.random() < 0.3 else 1000
        d = rng.integers(1, hi, size=rng.integers(0, 64)).astype(np.uint32)
        exact = sum((Fraction(1.0 / float(x)) for x in d), Fraction(0))
        assert oracle_port.exact_sum_recip(d) == float(exact)


def test_spec_examples(oracle_port):
    tri = CompressedCsr.from_adjacency([[1, 2], [0, 2], [0, 1]])
    m = oracle_port.local_metrics(tri)
    assert np.all(m["clustering"] == 1.0)
    star = CompressedCsr.from_adjacency([[1, 2, 3, 4, 5], [0], [0], [0], [0], [0]])
    m = oracle_port.local_metrics(star)
    assert m["control"][0] == 5.0 and np.all(m["control"][1:] == 0.2)
    assert m["controllability"][0] == 1.0 and np.all(m["controllability"][1:] == 0.2)
    assert m["clustering"][0] == 0.0 and np.all(np.isnan(m["clustering"][1:]))


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_random_gnp_vs_matrix_oracle(oracle_port, seed):
    A, g = random_graph(30, 0.3, seed)
    m = oracle_port.local_metrics(g)
    b = brute(A)
    for k in b:
        assert same(m[k], b[k]), k


def test_isolated_and_subrange(oracle_port):
    g = CompressedCsr.from_adjacency([[1], [0, 2], [1], [], [5], [4]])
    full = oracle_port.local_metrics(g)
    assert full["control"][3] == 0.0 and np.isnan(full["controllability"][3]) and np.isnan(full["clustering"][3])
    part = oracle_port.local_metrics(g, 2, 5)
    for k in full:
        assert same(part[k], full[k][2:5]), k


# ------------------------------------------------------------------ GPU parity
def graphs():
    yield "triangle", CompressedCsr.from_adjacency([[1, 2], [0, 2], [0, 1]])
    yield "star", CompressedCsr.from_adjacency([[1, 2, 3, 4, 5], [0], [0], [0], [0], [0]])
    yield "isolated", CompressedCsr.from_adjacency([[1], [0, 2], [1], [], [5], [4], []])
    for s in range(3):
        yield f"gnp{s}", random_graph(30, 0.3, s)[1]
    yield "gnp200", random_graph(200, 0.08, 11)[1]
    yield "c1like", CompressedCsr.synth_grid(32, 32, 8, 2, 5, 20261017, 0)
    yield "radius", CompressedCsr.synth_grid(40, 50, 12, 2, 6, 3, 9 * 9)
    yield "open", CompressedCsr.synth_grid(30, 30, 0, 1, 1, 1, 6 * 6)


@pytest.mark.gpu
@pytest.mark.parametrize("name,g", list(graphs()), ids=[n for n, _ in graphs()])
def test_gpu_local_metrics_bit_exact(oracle_port, name, g):
    ref = oracle_port.local_metrics(g)
    got = DeviceGraph(g).local_metrics()
    for k in ref:
        assert same(got[k], ref[k]), (name, k)


@pytest.mark.gpu
def test_gpu_local_metrics_subranges(oracle_port):
    g = CompressedCsr.synth_grid(24, 24, 6, 2, 5, 9, 0)
    ref = oracle_port.local_metrics(g)
    dg = DeviceGraph(g)
    n = g.n
    for v0, v1 in ((0, 1), (5, n // 3), (n // 3, n), (n - 1, n), (7, 7)):
        got = dg.local_metrics(v0, v1)
        for k in ref:
            assert same(got[k], ref[k][v0:v1]), (v0, v1, k)


@pytest.mark.gpu
def test_gpu_local_metrics_needs_full_graph():
    g = CompressedCsr.synth_grid(16, 16, 0, 1, 1, 1, 0)
    with pytest.raises(ValueError):
        DeviceGraph(g, node_range=(0, g.n // 2)).local_metrics()


@pytest.mark.gpu
@pytest.mark.parametrize("n2", ["bfs", "bitmap"])
@pytest.mark.parametrize("scratch", ["smem", "global"])
def test_gpu_local_metrics_both_n2_methods(n2, scratch):
    """|N2(v)| from the depth-2 BFS or from per-node 2-hop bitmaps (SB_LOCAL_N2), with the
    bitmaps in shared memory or in the per-CTA global scratch (SB_LOCAL_GLOBAL=1)."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np, oracle\n"
        "from paper_2604_08374_b200 import CompressedCsr, DeviceGraph\n"
        "from tests.test_local_metrics import random_graph\n"
        "for g in (CompressedCsr.synth_grid(32, 32, 8, 2, 5, 20261017, 0),\n"
        "          CompressedCsr.synth_grid(60, 70, 40, 1, 5, 9, 7 * 7), random_graph(120, 0.05, 3)[1],\n"
        "          CompressedCsr.from_adjacency([[1], [0, 2], [1], [], [5], [4], []])):\n"
        "    ref = oracle.port().local_metrics(g); got = DeviceGraph(g).local_metrics()\n"
        "    assert all(np.array_equal(got[k], ref[k], equal_nan=got[k].dtype.kind == 'f') for k in ref)\n"
        "print('ok')\n" % ROOT)
    env = dict(os.environ, SB_LOCAL_N2=n2, SB_LOCAL_GLOBAL="1" if scratch == "global" else "0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300,
                       cwd=ROOT)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


@pytest.mark.gpu
def test_gpu_local_metrics_hilbert_equivariant(tmp_path):
    """Renumbering permutes the exact local metrics and nothing else;
    also through a VGACSR03 save/load round trip."""
    g = CompressedCsr.synth_grid(40, 44, 14, 2, 6, 12, 9 * 9)
    h = g.hilbert_reorder()
    path = str(tmp_path / "h.vgacsr")
    h.save_vgacsr(path)
    h2 = CompressedCsr.load_vgacsr(path)
    inv = h.hilbert_inverse.astype(np.int64)
    ref = DeviceGraph(g).local_metrics()
    for hh in (h, h2):
        got = DeviceGraph(hh).local_metrics()
        for k in ref:
            assert same(got[k], ref[k][inv]), k


@pytest.mark.gpu
@pytest.mark.parametrize("n2", ["bfs", "bitmap"])
def test_gpu_local_metrics_wide_windows_paths_agree(tmp_path, n2):
    """A wide grid (raster ids make the per-node windows span whole grid rows): the
    1024-thread shared-memory path and the 256-thread global-scratch path agree."""
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from paper_2604_08374_b200 import DeviceGraph, grid_mask\n"
        "dg = DeviceGraph.from_grid(grid_mask(40, 4000, 300, 2, 6, 5), 30 * 30)\n"
        "m = dg.local_metrics(0, 4000)\n"
        "np.savez(sys.argv[1], **m)\n" % ROOT)
    outs = []
    for glob in ("0", "1"):
        f = str(tmp_path / f"m{glob}.npz")
        env = dict(os.environ, SB_LOCAL_N2=n2, SB_LOCAL_GLOBAL=glob)
        r = subprocess.run([sys.executable, "-c", code, f], env=env, capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(f))
    for k in outs[0].files:
        assert same(outs[0][k], outs[1][k]), k

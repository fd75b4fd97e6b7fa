"""On-device grid visibility graph construction (sb_graph_build_grid) vs the
host generator (sb_csr_synth_grid): byte-identical CSR, components and cell map."""
import numpy as np
import pytest

from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, HyperBall, grid_mask

CASES = [
    # rows, cols, rects, rmin, rmax, seed, radius2
    (32, 32, 8, 2, 5, 20261017, 0),
    (64, 64, 20, 2, 9, 20261017, 0),
    (40, 50, 12, 2, 6, 3, 9 * 9),
    (30, 30, 0, 1, 1, 1, 6 * 6),
    (1, 200, 0, 1, 1, 1, 0),
    (150, 1, 0, 1, 1, 1, 7),
    (1, 1, 0, 1, 1, 1, 0),
    (45, 300, 60, 1, 12, 9, 13 * 13),
    (25, 25, 40, 1, 4, 77, 2),
    (60, 60, 90, 1, 3, 5, 0),  # many small components
]


def test_grid_mask_matches_generator():
    for rows, cols, k, a, b, seed, _ in CASES[:4]:
        m = grid_mask(rows, cols, k, a, b, seed)
        g = CompressedCsr.synth_grid(rows, cols, k, a, b, seed, 0)
        free = np.nonzero(m.ravel() == 0)[0]
        assert np.array_equal(free.astype(np.uint32), g.cell_of_node)


@pytest.mark.gpu
@pytest.mark.parametrize("case", CASES, ids=[f"{c[0]}x{c[1]}r{c[6]}" for c in CASES])
def test_gpu_build_is_byte_identical(case):
    rows, cols, k, a, b, seed, r2 = case
    ref = CompressedCsr.synth_grid(rows, cols, k, a, b, seed, r2)
    dg = DeviceGraph.from_grid(grid_mask(rows, cols, k, a, b, seed), r2)
    assert dg.n == ref.n and dg.edges == ref.edges
    off, deg, st = dg.download()
    assert np.array_equal(off, ref.offsets)
    assert np.array_equal(deg, ref.degrees)
    assert np.array_equal(st, ref.stream)
    gi = dg.grid_info()
    assert (gi["rows"], gi["cols"]) == (rows, cols)
    assert np.array_equal(gi["cell_of_node"], ref.cell_of_node)
    assert np.array_equal(gi["component_id"], ref.component_id)
    assert np.array_equal(gi["component_sizes"], ref.component_sizes)


@pytest.mark.gpu
def test_gpu_build_large_components():
    """Union-find at scale (the flatten/label race shows up only on big graphs)."""
    for rows, cols, k, a, b, seed, r2 in ((300, 300, 0, 1, 1, 1, 20 * 20), (300, 300, 400, 1, 6, 4, 12 * 12)):
        ref = CompressedCsr.synth_grid(rows, cols, k, a, b, seed, r2)
        gi = DeviceGraph.from_grid(grid_mask(rows, cols, k, a, b, seed), r2).grid_info()
        assert np.array_equal(gi["component_id"], ref.component_id)
        assert np.array_equal(gi["component_sizes"], ref.component_sizes)


@pytest.mark.gpu
def test_gpu_build_errors():
    with pytest.raises(RuntimeError):
        DeviceGraph.from_grid(np.ones((4, 4), np.uint8))
    with pytest.raises(ValueError):
        DeviceGraph.from_grid(np.zeros(5, np.uint8))


@pytest.mark.gpu
def test_gpu_hyperball_on_device_built_graph():
    rows, cols, k, a, b, seed, r2 = 48, 48, 14, 2, 6, 11, 10 * 10
    ref = CompressedCsr.synth_grid(rows, cols, k, a, b, seed, r2)
    h1 = HyperBall(ref, 10)
    h1.run()
    dg = DeviceGraph.from_grid(grid_mask(rows, cols, k, a, b, seed), r2)
    h2 = HyperBall(dg, 10)
    h2.run()
    assert np.array_equal(h1.registers(), h2.registers())
    assert np.array_equal(h1.state().sum_d, h2.state().sum_d)
    assert np.array_equal(dg.node_count_of_component(), ref.node_count_of_component())
    assert np.array_equal(dg.local_metrics()["clustering"], DeviceGraph(ref).local_metrics()["clustering"],
                          equal_nan=True)

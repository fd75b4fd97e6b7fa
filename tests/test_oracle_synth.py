"""The oracle's benchmark-graph generator (oracle/sb_synth.c) vs the product's
(sb_csr_synth_grid): byte-identical offsets, degrees and stream, so the
reference arm of bench.py builds its input without mapping the product library."""
import hashlib
import json
import os

import numpy as np
import pytest

import oracle
from paper_2604_08374_b200 import CompressedCsr

CASES = [
    (64, 64, 20, 2, 9, 20261017, 0),              # C1
    (212, 212, 60, 3, 10, 20261017, 44 * 44),     # C2
    (30, 40, 7, 1, 5, 3, 9 * 9),
    (5, 7, 0, 1, 1, 1, 0),
    (1, 50, 3, 1, 2, 9, 0),
    (41, 3, 12, 1, 4, 77, 2),
]


@pytest.mark.parametrize("args", CASES, ids=[f"{a[0]}x{a[1]}r{a[2]}R{a[6]}" for a in CASES])
def test_oracle_generator_byte_identical(args):
    a = oracle.SynthCsr(*args)
    b = CompressedCsr.synth_grid(*args)
    assert a.n == b.n and a.edges == b.edges and a.stream_len == b.stream_len
    assert np.array_equal(a.offsets, b.offsets)
    assert np.array_equal(a.degrees, b.degrees)
    assert np.array_equal(a.stream, b.stream)


def test_oracle_generator_c3_matches_committed_hashes():
    """C3 (486^2, radius 87: 4.79e9 edges) -- hashes recorded from the product
    generator when the reference-path goldens were made."""
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "scale_reference.json")))["c3_p10"]["graph"]
    g = oracle.SynthCsr(486, 486, 0, 1, 1, 20261017, 87 * 87)
    assert (g.n, g.edges, g.stream_len) == (gold["nodes"], gold["edges"], gold["stream_bytes"])
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(g.offsets) == gold["offsets_sha256"] and sha(g.degrees) == gold["degrees_sha256"]
    assert hashlib.sha256(g.stream.data).hexdigest() == gold["stream_sha256"]

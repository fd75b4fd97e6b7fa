"""Generates tests/golden/scale_reference.json: per-iteration hashes of the
REFERENCE CPU path (oracle/_ref: the reference's own compiled hll/kernels
primitives + the SPEC loop of ref_shim.cpp) on BASELINE configs too large to
run in lockstep inside the GPU test session.

    python tests/golden/make_scale_golden.py c3          # ~6 min on 8 cores
    python tests/golden/make_scale_golden.py c2:4 c2:6   # C4 points (p sweep on C2)

Each case records, after EVERY iteration t: SHA-256 of the full register plane
(reference packed layout, hll.hpp:31-32), the max increase (f64 hex), and
SHA-256 of c_t, sum_d and sum_d2 (f64 arrays, little endian).  The graph is
the bench generator's (bench.CONFIGS); its offsets / degrees / stream hashes
are recorded too so a generator change cannot silently change the input.
"""
from __future__ import annotations

import hashlib
import json
import os
import struct
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import oracle  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "scale_reference.json")


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def graph_hashes(g) -> dict:
    return dict(nodes=int(g.n), edges=int(g.edges), stream_bytes=int(g.stream_len),
                offsets_sha256=sha(g.offsets), degrees_sha256=sha(g.degrees),
                stream_sha256=hashlib.sha256(g.stream_padded()[: g.stream_len].tobytes()).hexdigest())


def run_case(cfg: str, p: int, depth: int | None) -> dict:
    from bench import build_graph
    O = oracle.reference()
    g = build_graph(cfg, threads=os.cpu_count() or 1)
    t0 = time.perf_counter()
    rows = []

    def per_iter(t, regs, c):
        rows.append(dict(t=t, registers_sha256=sha(regs), c_sha256=sha(c)))

    r = O.hb_run(g, p, depth_limit=depth, threads=os.cpu_count() or 1, per_iteration=per_iter)
    for row, mx in zip(rows, r["max_increase"]):
        row["max_increase"] = struct.pack("<d", mx).hex()
    return dict(config=cfg, p=p, depth=depth, graph=graph_hashes(g), oracle=O.kind, ops=O._opsname().decode(),
                iterations=r["iterations"], converged=r["converged"], per_iteration=rows,
                sum_d_sha256=sha(r["sum_d"]), sum_d2_sha256=sha(r["sum_d2"]), c_sha256=sha(r["c"]),
                cpu_seconds=round(time.perf_counter() - t0, 1), cpu_threads=os.cpu_count())


def main(argv):
    if not oracle.reference_available():
        sys.exit("oracle/_ref/libsbref.so missing: run make -C oracle in the build container")
    data = json.load(open(OUT)) if os.path.exists(OUT) else {}
    for spec in argv or ["c3"]:
        cfg, _, rest = spec.partition(":")
        p, _, d = rest.partition(":")
        p = int(p or 10)
        depth = int(d) if d else None
        key = f"{cfg}_p{p}" + (f"_d{depth}" if depth else "")
        print(f"[golden] {key} ...", file=sys.stderr, flush=True)
        data[key] = run_case(cfg, p, depth)
        print(f"[golden] {key}: {data[key]['iterations']} iterations, {data[key]['cpu_seconds']} s",
              file=sys.stderr, flush=True)
        with open(OUT, "w") as f:
            json.dump(data, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:])

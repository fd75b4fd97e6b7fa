"""Upload-time stream validation (build_items_kernel) against a Python restatement.

The device validates every row once at upload (leb128.hpp:28-39,
restricted to 32-bit ids): varints of at most 5 bytes holding < 2^32, the first
id absolute and every later delta >= 1, ids < N without 32-bit wrap, exactly
deg ids per row and no trailing bytes.  Random valid graphs (rows up to ~1500
ids, so rows are cut into several work items) are mutated (byte flips, byte
values, truncation, insertion, degree and offset changes); the device must
accept exactly the streams `valid_rows` accepts, for the synchronous and the
asynchronous upload.  Accepted mutants must also run HyperBall bit-exactly
against the oracle (so the work items and the longest-run bound were right).
"""
import numpy as np
import pytest

import oracle

from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, HyperBall
from paper_2604_08374_b200.cgraph import encode_neighbor_row


def valid_rows(n, offsets, degrees, stream):
    for v in range(n):
        pos, end = int(offsets[v]), int(offsets[v + 1])
        if end < pos:
            return False
        prev = None
        for _ in range(int(degrees[v])):
            val, shift, k = 0, 0, 0
            while True:
                if pos >= end:
                    return False  # truncated
                b = int(stream[pos])
                pos += 1
                val |= (b & 0x7F) << shift
                shift += 7
                k += 1
                if not b & 0x80:
                    break
                if k == 5:
                    return False  # > 5 bytes
            if val >= 2**32:
                return False
            x = val if prev is None else prev + val
            if prev is not None and val == 0:
                return False
            if x >= n or x >= 2**32:
                return False
            prev = x
        if pos != end:
            return False  # trailing bytes
    return True


def random_graph(rng):
    n = int(rng.integers(2, 1700))
    rows = []
    for v in range(n):
        r = rng.random()
        if r < 0.15:
            d = 0
        elif r < 0.25:
            d = int(rng.integers(500, min(n, 1600) + 1)) if n > 500 else int(rng.integers(0, n + 1))
        else:
            d = int(rng.integers(0, min(n, 40) + 1))
        ids = np.sort(rng.choice(n, size=d, replace=False)) if d else np.zeros(0, np.int64)
        if d and rng.random() < 0.5:  # long runs of consecutive ids
            s = int(rng.integers(0, n - d + 1))
            ids = np.arange(s, s + d)
        rows.append(ids)
    enc = [encode_neighbor_row(r.tolist()) for r in rows]
    off = np.zeros(n + 1, np.uint64)
    off[1:] = np.cumsum([len(e) for e in enc])
    deg = np.array([len(r) for r in rows], np.uint32)
    stream = np.frombuffer(b"".join(enc), np.uint8).copy()
    return n, off, deg, stream


def mutate(rng, n, off, deg, stream):
    off, deg, stream = off.copy(), deg.copy(), stream.copy()
    kind = int(rng.integers(0, 8))
    nz = np.nonzero(np.diff(off.astype(np.int64)))[0]
    if kind == 0 and len(stream):  # flip the continuation bit of one byte
        i = int(rng.integers(0, len(stream)))
        stream[i] ^= 0x80
    elif kind == 1 and len(stream):  # random byte value
        stream[int(rng.integers(0, len(stream)))] = int(rng.integers(0, 256))
    elif kind == 2 and len(nz):  # drop the last byte of a row (shift later offsets)
        v = int(rng.choice(nz))
        cut = int(off[v + 1]) - 1
        stream = np.delete(stream, cut)
        off[v + 1:] -= 1
    elif kind == 3 and len(nz):  # insert a byte into a row
        v = int(rng.choice(nz))
        at = int(rng.integers(int(off[v]), int(off[v + 1]) + 1))
        stream = np.insert(stream, at, np.uint8(rng.integers(0, 256)))
        off[v + 1:] += 1
    elif kind == 4:  # degree off by one
        v = int(rng.integers(0, n))
        deg[v] = max(0, int(deg[v]) + int(rng.choice([-1, 1])))
    elif kind == 5 and len(nz):  # overlong first id (5-byte varint with a large top byte)
        v = int(rng.choice(nz))
        a = int(off[v])
        if stream[a] < 0x80:
            top = int(rng.integers(0, 0x80))
            ins = np.array([stream[a] | 0x80, 0x80, 0x80, 0x80, top], np.uint8)
            stream = np.concatenate([stream[:a], ins, stream[a + 1:]])
            off[v + 1:] += 4
    elif kind == 6 and len(nz):  # zero delta (repeat) at a random position of a row
        v = int(rng.choice(nz))
        at = int(off[v + 1])
        stream = np.insert(stream, at, np.uint8(0))
        off[v + 1:] += 1
        deg[v] += 1
    elif kind == 7 and len(nz):  # huge delta that wraps 32 bits
        v = int(rng.choice(nz))
        at = int(off[v + 1])
        big = np.frombuffer(bytes([0xFF, 0xFF, 0xFF, 0xFF, 0x0F]), np.uint8)
        stream = np.insert(stream, at, big)
        off[v + 1:] += 5
        deg[v] += 1
    return off, deg, stream


def device_accepts(n, off, deg, stream, async_upload):
    try:
        if async_upload:
            csr = CompressedCsr.from_arrays(off, deg, stream)
            dg = DeviceGraph(csr, async_upload=True)
            dg.wait()
        else:
            DeviceGraph.from_raw(n, off, deg, stream)
        return True
    except RuntimeError:
        return False


def test_python_validator_accepts_encoder_output():
    rng = np.random.default_rng(5)
    for _ in range(20):
        assert valid_rows(*random_graph(rng))


@pytest.mark.gpu
@pytest.mark.parametrize("seed", range(4))
def test_gpu_validation_matches_python(seed, oracle_best):
    rng = np.random.default_rng(1000 + seed)
    agree = accepted_mutants = rejected = 0
    for case in range(60):
        n, off, deg, stream = random_graph(rng)
        if case % 3:
            off, deg, stream = mutate(rng, n, off, deg, stream)
        expect = valid_rows(n, off, deg, stream)
        got = device_accepts(n, off, deg, stream, async_upload=False)
        assert got == expect, (seed, case)
        agree += 1
        rejected += not expect
        if expect:
            accepted_mutants += case % 3 != 0
            csr = CompressedCsr.from_arrays(off, deg, stream)
            hb = HyperBall(csr, 10, 3)
            hb.run()
            ref = oracle_best.hb_run(csr, 10, 3)
            assert np.array_equal(hb.registers(), ref["registers"]), (seed, case)
            assert np.array_equal(hb.state().sum_d, ref["sum_d"]), (seed, case)
            # the run index (interval mode, local metrics) over the same rows and work items
            hi = HyperBall(csr, 10, 3, interval=True)
            hi.run()
            assert np.array_equal(hi.registers(), ref["registers"]), (seed, case)
            if case % 4 == 0:
                lm = DeviceGraph(csr).local_metrics()
                lo = oracle.port().local_metrics(csr)
                for k in lo:
                    assert np.array_equal(lm[k], lo[k], equal_nan=lm[k].dtype.kind == "f"), (seed, case, k)
    assert rejected > 10


@pytest.mark.gpu
def test_gpu_validation_async_matches_python():
    rng = np.random.default_rng(77)
    for case in range(40):
        n, off, deg, stream = random_graph(rng)
        off, deg, stream = mutate(rng, n, off, deg, stream)
        if int(off[-1]) != len(stream):
            continue
        expect = valid_rows(n, off, deg, stream)
        try:
            CompressedCsr.from_arrays(off, deg, stream)
        except RuntimeError:
            continue  # the host loader already refuses it
        assert device_accepts(n, off, deg, stream, async_upload=True) == expect, case

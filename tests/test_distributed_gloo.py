"""N>1 host path on CPU: world_size-2 (and 3) gloo process groups.

The device exchange is NCCL inside libsieveball_cuda (untestable without
GPUs); what is tested here is everything around it with the same semantics:
edge-balanced shard bounds agree on every rank, each rank computes only its
range against the full replica, the shard rows are exchanged (here with
gloo broadcasts mirroring the grouped ncclBroadcast), the max increase is
all-reduced before the convergence test, and the result gathered on rank 0
is bit-identical to a single-process run (SPEC.md:451 determinism regardless
of worker count).
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2604_08374_b200 import CompressedCsr
        from paper_2604_08374_b200.distributed import gather_to_root, shard_bounds
        O = oracle.port()
        g = CompressedCsr.synth_grid(24, 24, 8, 2, 5, 17, 0)
        p = 8
        b = shard_bounds(g, world)
        allb = [None] * world
        dist.all_gather_object(allb, b.tolist())
        assert all(x == b.tolist() for x in allb)
        v0, v1 = int(b[rank]), int(b[rank + 1])
        rb = (1 << p) // 2
        cur, c_prev = O.hb_init(g.n, p)
        nxt = np.zeros_like(cur)
        c_cur, sd, sd2 = np.zeros(g.n), np.zeros(g.n), np.zeros(g.n)
        t = 0
        while True:
            t += 1
            local = O.hb_iterate(g, p, t, cur, nxt, c_prev, c_cur, sd, sd2, v0=v0, v1=v1, threads=1)
            # exchange: every shard broadcasts its rows (== grouped ncclBroadcast)
            for r in range(world):
                a, e = int(b[r]), int(b[r + 1])
                if e > a:
                    buf = torch.from_numpy(nxt[a * rb:e * rb].copy())
                    dist.broadcast(buf, src=r)
                    nxt[a * rb:e * rb] = buf.numpy()
            mx = torch.tensor([local], dtype=torch.float64)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)  # == ncclAllReduce(max)
            if mx.item() <= 0.5:
                break
            cur, nxt = nxt, cur
            c_prev, c_cur = c_cur, c_prev
        full = gather_to_root(sd[v0:v1].copy(), b, rank, world)
        if rank == 0:
            ref = O.hb_run(g, p)
            q.put((t == ref["iterations"], bool(np.array_equal(full, ref["sum_d"])),
                   bool(np.array_equal(nxt, ref["registers"]))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_hyperball_gloo_bit_identical(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    same_t, same_sum, same_regs = q.get(timeout=5)
    assert same_t and same_sum and same_regs


def _p2p_fallback_worker(rank, world, port, fail_rank, q):
    """sharded_hyperball's agreement on the exchange: one rank's CUDA IPC attach
    fails -> every rank ends on the grouped-broadcast exchange, and ranks whose
    attach had succeeded rebuild their state without peers."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2604_08374_b200.distributed as D
        from paper_2604_08374_b200 import CompressedCsr
        made = []

        class FakeHB:
            def __init__(self, *a, **k):
                self.peers = False
                self.closed = False
                made.append(self)

            def close(self):
                self.closed = True

        def fake_attach(hb, r, w, b):
            if r == fail_rank:
                raise RuntimeError("cudaIpcOpenMemHandle: peer access not supported")
            hb.peers = True

        D.HyperBall, D.DeviceGraph, D.attach_peers = FakeHB, (lambda *a, **k: None), fake_attach
        g = CompressedCsr.synth_grid(12, 12, 0, 1, 1, 1, 0)
        hb = D.sharded_hyperball(g, 10, None, rank, world, 0, None)
        q.put((rank, hb.exchange_mode, hb.peers, len(made), made[0].closed))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("fail_rank", [1, None])
def test_fused_p2p_fallback_agreement(fail_rank):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    world = 3
    procs = [ctx.Process(target=_p2p_fallback_worker, args=(r, world, port, fail_rank, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    for pr in procs:
        pr.join(timeout=240)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    res = sorted(q.get(timeout=5) for _ in range(world))
    for rank, mode, peers, n_made, first_closed in res:
        if fail_rank is None:
            assert mode == "fused-p2p" and peers and n_made == 1
        else:
            assert mode.startswith("nccl-broadcast (fused P2P unavailable: RuntimeError: cudaIpcOpenMemHandle")
            assert not peers
            assert n_made == (1 if rank == fail_rank else 2) and first_closed == (rank != fail_rank)

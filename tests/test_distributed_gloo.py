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

"""Multi-rank NCCL exchange inside libsieveball_cuda (one process per rank).

Each rank owns an edge-balanced node range, computes only that range, and
sb_hb_step exchanges the new rows with grouped ncclBroadcast and the max
increase with ncclAllReduce.  The gathered result must be bit-identical to a
single-GPU run.  Ranks are placed on distinct GPUs when available; with one
GPU they share device 0 (NCCL may refuse duplicate devices -- then the test
skips with NCCL's message).
"""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank(rank, world, port, q, interval):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import torch
        from paper_2604_08374_b200 import CompressedCsr, HyperBall
        from paper_2604_08374_b200.distributed import gather_to_root, init_comm, sharded_hyperball, shard_bounds
        ndev = torch.cuda.device_count()
        dev = rank % ndev
        g = CompressedCsr.synth_grid(64, 64, 20, 2, 9, 20261017, 0)
        b = shard_bounds(g, world)
        try:
            comm = init_comm(rank, world, dev)
        except Exception as e:  # NCCL refuses duplicate GPUs on some versions
            q.put(("skip", f"{type(e).__name__}: {e}"))
            return
        hb = sharded_hyperball(g, 10, None, rank, world, dev, comm, bounds=b, interval=interval)
        it = hb.run()
        st = hb.state()
        sd = gather_to_root(st.sum_d, b, rank, world)
        regs = hb.registers()
        xs = [s["exchange_ms"] for s in hb.stats()]
        if rank == 0:
            ref = HyperBall(g, 10, None, device=dev)
            ref.run()
            rs = ref.state(with_registers=True)
            q.put(("ok", it == rs.t, bool(np.array_equal(sd, rs.sum_d)),
                   bool(np.array_equal(regs, rs.registers)), max(xs)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,interval", [(2, False), (2, True), (3, False)])
def test_nccl_sharded_bit_identical(world, interval):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank, args=(r, world, port, q, interval)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    for p in ps:
        if p.is_alive():
            p.kill()
    res = q.get(timeout=10)
    if res[0] == "skip":
        pytest.skip("NCCL multi-rank on this box: " + res[1])
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    _, same_t, same_sum, same_regs, xms = res
    assert same_t and same_sum and same_regs
    assert xms > 0.0  # the exchange actually ran


@pytest.mark.parametrize("interval", [False, True])
def test_nccl_exchange_one_rank_communicator(interval):
    """The in-library exchange (grouped ncclBroadcast of the shard rows + 8-byte
    ncclAllReduce(max), sb_hb_api.cu exchange_nccl) runs for ANY attached
    communicator, a 1-rank one included, so it executes on a 1-GPU box: every
    iteration goes through it and the result stays bit-identical."""
    from paper_2604_08374_b200 import CompressedCsr, HyperBall
    from paper_2604_08374_b200.hyperball import Comm
    g = CompressedCsr.synth_grid(64, 64, 20, 2, 9, 20261017, 0)
    ref = HyperBall(g, 10, None, interval=interval)
    ref.run()
    comm = Comm(1, 0, Comm.unique_id(), 0)
    hb = HyperBall(g, 10, None, interval=interval)
    hb.attach_comm(comm, [0, g.n])
    for _ in range(2):  # run, reset, run again
        hb.run()
        st = hb.stats()
        assert len(st) == ref.t and all(s["exchange_ms"] > 0.0 for s in st)
        assert np.array_equal(hb.registers(), ref.registers())
        assert np.array_equal(hb.state().sum_d, ref.state().sum_d)
        hb.reset()
    del hb
    comm.close()


def _rank_p2p(rank, world, port, q, mode):
    """Two+ processes, fused P2P row stores over CUDA IPC, gloo barrier + max."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2604_08374_b200 import CompressedCsr, HyperBall
        from paper_2604_08374_b200.distributed import attach_peers, gather_to_root, shard_bounds
        dev = rank % torch.cuda.device_count()
        g = CompressedCsr.synth_grid(64, 64, 20, 2, 9, 20261017, 0)
        b = shard_bounds(g, world)
        hb = HyperBall(g, 10, None, device=dev, node_range=(int(b[rank]), int(b[rank + 1])),
                       skip_unchanged=(mode == "skip"), interval=(mode == "interval"))
        attach_peers(hb, rank, world, b)
        while True:
            mx = torch.tensor([hb.step_compute()], dtype=torch.float64)
            dist.all_reduce(mx, op=dist.ReduceOp.MAX)  # barrier: every rank's rows are pushed
            if hb.step_finish(mx.item())[1]:
                break
        sd = gather_to_root(hb.state().sum_d, b, rank, world)
        regs = hb.registers()
        if rank == 0:
            ref = HyperBall(g, 10, None, device=dev)
            ref.run()
            rs = ref.state(with_registers=True)
            q.put((hb.t == rs.t, bool(np.array_equal(sd, rs.sum_d)), bool(np.array_equal(regs, rs.registers))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode", [(2, "dense"), (3, "dense"), (2, "skip"), (2, "interval")])
def test_fused_p2p_exchange_bit_identical(world, mode):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_p2p, args=(r, world, port, q, mode)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    for p in ps:
        if p.is_alive():
            p.kill()
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    same_t, same_sum, same_regs = q.get(timeout=10)
    assert same_t and same_sum and same_regs


def _rank_widened(rank, world, port, q):
    """Local metrics by node range and exact BFS by source range, summed over gloo."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    import traceback
    import torch
    import torch.distributed as dist
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        _widened_body(rank, world, q, torch, dist)
    except Exception:
        q.put(("error", rank, traceback.format_exc()))
        raise
    finally:
        dist.destroy_process_group()


def _widened_body(rank, world, q, torch, dist):
    if True:
        from paper_2604_08374_b200 import CompressedCsr, DeviceGraph, exact_bfs_all
        from paper_2604_08374_b200.distributed import (gather_to_root, shard_bounds, sharded_exact_bfs,
                                                       sharded_local_metrics)
        dev = rank % torch.cuda.device_count()
        g = CompressedCsr.synth_grid(90, 100, 30, 2, 6, 21, 9 * 9)  # > 8192 nodes: 3 source blocks
        b = shard_bounds(g, world)
        lm = sharded_local_metrics(g, rank, world, dev, b)
        clus = gather_to_root(lm["clustering"], b, rank, world)
        ex = sharded_exact_bfs(g, rank, world, dev)
        tot = {}
        for k in ("sum_d", "sum_d2", "reach"):
            t = torch.from_numpy(ex[k].astype(np.int64))
            dist.all_reduce(t)
            tot[k] = t.numpy()
        if rank == 0:
            ref_l = DeviceGraph(g).local_metrics()["clustering"]
            ref_x = exact_bfs_all(g)
            q.put(("ok", bool(np.array_equal(clus, ref_l, equal_nan=True)),
                   all(bool(np.array_equal(tot[k], ref_x[k].astype(np.int64))) for k in tot)))


@pytest.mark.parametrize("world", [2, 3])
def test_widened_passes_shard_without_exchange(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    ps = [ctx.Process(target=_rank_widened, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    for p in ps:
        p.join(timeout=300)
    for p in ps:
        if p.is_alive():
            p.kill()
    res = q.get(timeout=10)
    assert res[0] == "ok", res
    assert all(p.exitcode == 0 for p in ps), [p.exitcode for p in ps]
    assert res[1] and res[2]

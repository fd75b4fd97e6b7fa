"""Node-range sharding across GPUs (one process per GPU).

The reference parallelises iterate_once over contiguous node ranges inside one
process (parallel.hpp:20-47).  Here each rank owns a contiguous,
edge-balanced node range of the CSR in its own HBM plus a full replica of the
register plane; after every iteration the ranks exchange their freshly
computed rows (grouped NCCL broadcasts, one per shard, inside
libsieveball_cuda) and take the global max increase (NCCL all-reduce) before
the convergence test.  torch.distributed only bootstraps: it broadcasts the
NCCL unique id and gathers results for reporting.
"""
from __future__ import annotations

import numpy as np

from .cgraph import CompressedCsr
from .hyperball import Comm, DeviceGraph, HllParams, HyperBall


def shard_bounds(csr: CompressedCsr, world: int) -> np.ndarray:
    """Edge-balanced contiguous node ranges (bounds[world+1])."""
    return csr.partition(world)


def init_comm(rank: int, world: int, device: int) -> Comm | None:
    """NCCL communicator bootstrapped over the default torch.distributed group."""
    if world <= 1:
        return None
    import torch.distributed as dist
    uid = [Comm.unique_id() if rank == 0 else None]
    dist.broadcast_object_list(uid, src=0)
    return Comm(world, rank, uid[0], device)


def attach_peers(hb: HyperBall, rank: int, world: int, bounds: np.ndarray) -> None:
    """Fused P2P exchange: all-gather the CUDA IPC handles over torch.distributed
    and attach them, so the union kernel stores rows into every peer replica."""
    import torch.distributed as dist
    hs = [None] * world
    dist.all_gather_object(hs, hb.ipc_handles())
    hb.attach_peers(rank, hs, bounds)


def sharded_hyperball(csr: CompressedCsr, params: HllParams | int, depth_limit: int | None, rank: int,
                      world: int, device: int, comm: Comm | None, skip_unchanged: bool = False,
                      bounds: np.ndarray | None = None, interval: bool = False,
                      fused_p2p: bool = True, external_barrier: bool = False) -> HyperBall:
    """This rank's HyperBall over its node range, wired to the communicator.
    fused_p2p: rows travel as P2P stores from the union kernel (NCCL only
    carries the 8-byte max / barrier); otherwise grouped ncclBroadcast.
    external_barrier: no NCCL at all (ranks sharing a GPU): fused P2P rows, and
    the caller runs the iterations with run_external_barrier."""
    import os
    b = shard_bounds(csr, world) if bounds is None else bounds
    v0, v1 = int(b[rank]), int(b[rank + 1])

    def make():
        return HyperBall(DeviceGraph(csr, device, (v0, v1)), params, depth_limit, skip_unchanged=skip_unchanged,
                         interval=interval)

    hb = make()
    hb.exchange_mode = "single"
    if world > 1 and external_barrier:  # no NCCL (ranks share a device): fused P2P + external barrier only
        attach_peers(hb, rank, world, b)
        hb.exchange_mode = "fused-p2p (external torch.distributed barrier)"
        return hb
    if world > 1:
        hb.exchange_mode = "nccl-broadcast"
        if fused_p2p and os.environ.get("SB_P2P", "1") != "0":
            # Every rank must agree: a rank whose CUDA IPC attach fails (no peer
            # access, IPC blocked by the container) sends all ranks back to the
            # grouped-broadcast exchange.
            import torch.distributed as dist
            err = None
            try:
                attach_peers(hb, rank, world, b)
            except Exception as e:  # noqa: BLE001 -- reported, then agreed on
                err = f"{type(e).__name__}: {e}"
            errs = [None] * world
            dist.all_gather_object(errs, err)
            if any(errs):
                if err is None:  # peers attached here but not everywhere: start over without them
                    hb.close()
                    hb = make()
                hb.exchange_mode = "nccl-broadcast (fused P2P unavailable: " + next(e for e in errs if e) + ")"
            else:
                hb.exchange_mode = "fused-p2p"
    if comm is not None:
        hb.attach_comm(comm, b)
    return hb


def run_external_barrier(hb: HyperBall) -> int:
    """Alg. 1 for a rank whose rows travel as fused P2P stores but whose ranks
    share no NCCL communicator (e.g. several ranks on one GPU, which NCCL
    refuses): step_compute (returns after this rank's union kernel, and so its
    peer stores, completed), then a torch.distributed all-reduce of the local
    max increase -- the iteration barrier -- then step_finish."""
    import torch
    import torch.distributed as dist
    while True:
        mx = torch.tensor([hb.step_compute()], dtype=torch.float64)
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        if hb.step_finish(float(mx.item()))[1]:
            return hb.t


def reset_external_barrier(hb: HyperBall) -> None:
    """sb_hb_reset + the barrier that keeps peers from storing into a replica that
    is still being re-initialised (the in-library NCCL barrier's role)."""
    import torch.distributed as dist
    hb.reset()
    dist.barrier()


def gather_to_root(local: np.ndarray, bounds: np.ndarray, rank: int, world: int) -> np.ndarray | None:
    """Concatenate every rank's local-range array on rank 0 (node order)."""
    if world <= 1:
        return local
    import torch.distributed as dist
    parts = [None] * world if rank == 0 else None
    dist.gather_object(local, parts, dst=0)
    if rank != 0:
        return None
    out = np.concatenate(parts)
    assert out.shape[0] == int(bounds[-1])
    return out


def sharded_local_metrics(csr: CompressedCsr, rank: int, world: int, device: int,
                          bounds: np.ndarray | None = None) -> dict[str, np.ndarray]:
    """Exact local metrics for this rank's node range (no exchange: every rank
    holds the full CSR in its HBM; results concatenate in node order)."""
    b = shard_bounds(csr, world) if bounds is None else bounds
    return DeviceGraph(csr, device).local_metrics(int(b[rank]), int(b[rank + 1]))


def sharded_exact_bfs(csr: CompressedCsr, rank: int, world: int, device: int, depth_limit: int | None = None,
                      interval: bool = True) -> dict[str, np.ndarray]:
    """Exact BFS over this rank's share of the SOURCES (contiguous 4096-source
    blocks); per-node sum_d / sum_d2 / reach / histogram are partial sums that
    the caller adds across ranks (all_reduce(SUM)) -- no exchange during the run."""
    from .exact import ExactBfs
    blocks = (csr.n + 4095) // 4096
    b0, b1 = blocks * rank // world, blocks * (rank + 1) // world
    x = ExactBfs(csr, depth_limit, interval=interval, device=device)
    x.run(min(b0 * 4096, csr.n), min(b1 * 4096, csr.n))
    return x.result()

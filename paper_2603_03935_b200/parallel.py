"""Multi-GPU orchestration of the DISC path (one process per GPU, torch.distributed).

The map is key-hash sharded: rank r is shard r of G; it owns the voxel
keys with (mix64(key) >> 40) mod G == r and a replica of the instance table, runs stage 1 for the
stream's frames f = r + G j, and exchanges with the other ranks inside libdisc over NCCL (detection
records all-gathered and (s, key) pairs routed to their owners per window; partial overlap-count
triples all-gathered and new-membership counts all-reduced per frame).  This module only does the
host-side plumbing around it: process-group setup, the NCCL unique-id bootstrap (rank 0 creates it
with disc_nccl_unique_id, the process group broadcasts it), the frame split, barriers and
max-over-ranks timing.  Backend: NCCL when CUDA is available, gloo otherwise (CPU tests).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

SEED_STRIDE = 7919   # independent-map mode: rank r maps the stream with seed  base + SEED_STRIDE * r


@dataclass
class Rank:
    world: int
    rank: int
    local: int
    backend: str | None

    @property
    def distributed(self) -> bool:
        return self.world > 1


def setup(backend: str | None = None) -> Rank:
    """Initialise the process group from torchrun's environment (RANK, WORLD_SIZE, ...)."""
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws == 1:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
        return Rank(1, 0, 0, None)
    import torch.distributed as dist
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    if not dist.is_initialized():
        if backend == "nccl":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    return Rank(ws, rank, local, backend)


def sharded_map_kwargs(r: Rank) -> dict:
    """disc_config fields that make this process shard r.rank of an r.world-way key-sharded map:
    rank 0 creates the 128-byte NCCL unique id (disc_nccl_unique_id) and the process group
    broadcasts it, so every rank passes the same id (S:§8(b) bootstrap).  world 1: unsharded."""
    if not r.distributed:
        return dict(world_size=1, rank=0)
    import torch.distributed as dist
    obj = [None]
    if r.rank == 0:
        from .disc import nccl_unique_id
        obj[0] = nccl_unique_id()
    dist.broadcast_object_list(obj, src=0)
    return dict(world_size=r.world, rank=r.rank, nccl_unique_id=obj[0])


def own_frames(n: int, r: Rank) -> list:
    """Indices of the stream's first n frames that rank r integrates: f = r + G j (disc.h sharding)."""
    return list(range(r.rank, n, r.world))


def stream_seed(base: int, rank: int) -> int:
    return base + SEED_STRIDE * rank


def barrier(r: Rank) -> None:
    if r.distributed:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x: float, r: Rank) -> float:
    """Max of a scalar (device time) over ranks."""
    if not r.distributed:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", r.local) if r.backend == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float, r: Rank) -> float:
    if not r.distributed:
        return x
    import torch
    import torch.distributed as dist
    dev = torch.device("cuda", r.local) if r.backend == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def weak_scaling_rate(frames_per_rank: int, seconds: float, r: Rank) -> float:
    """Aggregate frames/s: every rank's frames over the slowest rank's time."""
    total = sum_over_ranks(float(frames_per_rank), r)
    return total / max_over_ranks(seconds, r)


def teardown(r: Rank) -> None:
    if r.distributed:
        import torch.distributed as dist
        if dist.is_initialized():
            dist.destroy_process_group()

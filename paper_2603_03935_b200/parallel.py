"""Multi-GPU orchestration of the DISC path (one process per GPU, torch.distributed).

This round the path scales as independent maps (SURVEY §8(e) frame-/scene-parallel stage):
every rank integrates its own scene stream (a rank-specific seed), there is no data-path
collective, and throughput is all frames processed / the max over ranks of the device time
(weak scaling).  The key-hash-sharded single map with NCCL all-to-all + allreduce is NEXT
(DESIGN.md §8).  Backend: NCCL when CUDA is available, gloo otherwise (CPU tests).
"""
from __future__ import annotations

import os
from dataclasses import dataclass

SEED_STRIDE = 7919   # rank r maps the stream with seed  base + SEED_STRIDE * r


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

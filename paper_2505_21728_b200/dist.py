"""Multi-GPU plumbing for the HyGT hot path.

Vectors are independent, so rows shard across ranks as contiguous ranges with
no data movement between GPUs; every rank holds a full plan replica (<= 1.2 MB of tables). The
only exchange step is the per-class per-coefficient energy sum of config 5: each rank's
forward kernel accumulates its shard's [C][N] fp64 sums (the fused epilogue), then one
all-reduce adds them (shards merge by addition, statistics.hpp:110-120). On B200 boxes the
collective runs over NCCL / NVLink; the same host logic runs over gloo in the CPU tests.
"""
from __future__ import annotations

import os
from typing import Optional, Tuple

import torch
import torch.distributed as dist


def _active(group=None) -> bool:
    return dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1


def init_process_group_from_env(device: Optional[torch.device] = None) -> Tuple[int, int]:
    """One process per GPU as torchrun launches it: join the NCCL group when WORLD_SIZE > 1
    (gloo for a CPU device). Returns (rank, world)."""
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world > 1 and not dist.is_initialized():
        if device is not None and device.type == "cuda":
            dist.init_process_group("nccl", device_id=device)
        else:
            dist.init_process_group("gloo")
    return rank, world


def destroy() -> None:
    if dist.is_available() and dist.is_initialized():
        dist.destroy_process_group()


def barrier(group=None) -> None:
    if _active(group):
        dist.barrier(group=group)


def sum_over_ranks(value: int, device=None, group=None) -> int:
    """Total units processed by all ranks (each rank's own count, so uneven shards add up)."""
    if not _active(group):
        return value
    t = torch.tensor([value], dtype=torch.int64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return int(t.item())


def shard_range(count: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous [begin, end) rows of `rank`; the shards partition [0, count) in rank order."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("shard_range: bad rank/world")
    base, extra = divmod(count, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def allreduce_energy(energy: torch.Tensor, group: Optional[dist.ProcessGroup] = None) -> torch.Tensor:
    """Sum the per-class energy accumulators of all ranks in place (fp64, [C][N])."""
    if energy.dtype != torch.float64:
        raise ValueError("allreduce_energy: energy must be float64")
    if _active(group):
        dist.all_reduce(energy, op=dist.ReduceOp.SUM, group=group)
    return energy


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Device-timed step durations are reported as the max over ranks."""
    if not _active(group):
        return value
    t = torch.tensor([value], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def sharded_forward_energy(plan, x_shard, cls_shard, energy, out=None, workspace=None, group=None):
    """Forward of this rank's rows plus the fused energy epilogue, then the energy all-reduce:
    on return every rank holds the energy of the whole (sharded) batch."""
    energy.zero_()
    y = plan.forward_energy(x_shard, cls_shard, energy, out=out, workspace=workspace)
    allreduce_energy(energy, group)
    return y


def allreduce_correlation(sums, counts, group=None):
    """Shards of the per-class second moments merge by addition (merge_correlation,
    statistics.hpp:110-120 weights by counts, which is the same as adding sums and counts)."""
    if _active(group):
        dist.all_reduce(sums, group=group)
        dist.all_reduce(counts, group=group)
    return sums, counts

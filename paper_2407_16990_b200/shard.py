"""Multi-GPU sharding of the hot path.

The path shards naturally: streams are independent and nothing crosses between them inside a step.
The unit of work is a *selection group* — `group` consecutive streams x one F-frame chunk, the scope
of the paper's cross-stream top-N ("aggregates and sorts MBs from all streams"). Groups are
assigned to ranks contiguously, so every group is computed by exactly one rank with the same inputs
whatever the world size, and the outputs are bit-identical for any world size. One process per
GPU; torch.distributed (NCCL on GPUs, gloo in the CPU tests) carries only the two reductions of the
measurement: MAX of the per-rank elapsed time and SUM of the frames processed.
"""
from __future__ import annotations


def group_bounds(n_streams: int, group: int) -> list[tuple[int, int]]:
    """[s0, s1) stream ranges of the selection groups (the last one may be short)."""
    if n_streams < 0 or group < 1:
        raise ValueError("n_streams >= 0 and group >= 1 required")
    return [(s, min(s + group, n_streams)) for s in range(0, n_streams, group)]


def rank_slice(n_items: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, balanced [i0, i1) share of `n_items` for `rank` (the first n % world ranks get one
    more)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("0 <= rank < world required")
    q, r = divmod(n_items, world)
    i0 = rank * q + min(rank, r)
    return i0, i0 + q + (1 if rank < r else 0)


def rank_groups(n_streams: int, group: int, world: int, rank: int) -> list[tuple[int, int]]:
    """The selection groups (stream ranges) rank `rank` of `world` processes."""
    gb = group_bounds(n_streams, group)
    g0, g1 = rank_slice(len(gb), world, rank)
    return gb[g0:g1]


def reduce_timing(elapsed_ms: float, frames: float, device=None) -> tuple[float, float]:
    """(MAX over ranks of elapsed_ms, SUM over ranks of frames); identity without a process group.
    `device` is where the reduction tensors live (cuda for NCCL, cpu for gloo)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(elapsed_ms), float(frames)
    t = torch.tensor([elapsed_ms], dtype=torch.float64, device=device)
    f = torch.tensor([frames], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dist.all_reduce(f, op=dist.ReduceOp.SUM)
    return float(t.item()), float(f.item())

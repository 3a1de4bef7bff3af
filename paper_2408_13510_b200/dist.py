"""Multi-GPU plumbing: replays shard across ranks with no data-path collective;
one final all-gather collects the fixed-size per-replay statistics records.

One process per GPU (torchrun), backend "nccl" on GPUs ("gloo" in the CPU
tests).  The replay kernels never communicate: a replay is an independent
unit, so rank r simply owns a contiguous block of seeds.
"""
from __future__ import annotations

import numpy as np

from . import abi


def shard_seeds(per_rank: int, rank: int, base: int = 1) -> np.ndarray:
    """Seeds of rank `rank` when every rank owns `per_rank` replays (weak
    scaling): rank r takes base + r*per_rank ... base + (r+1)*per_rank - 1."""
    start = base + rank * per_rank
    return np.arange(start, start + per_rank, dtype=np.uint64)


def split_seeds(seeds, rank: int, world: int) -> np.ndarray:
    """Strong-scaling split of a fixed seed list: contiguous, balanced blocks."""
    seeds = np.asarray(seeds, dtype=np.uint64)
    bounds = np.linspace(0, len(seeds), world + 1).astype(np.int64)
    return seeds[bounds[rank]:bounds[rank + 1]]


def gather_stats(stats_u8, world: int):
    """All-gather each rank's rs_replay_stats records (a uint8 tensor of
    256-byte records, equal length on every rank) in rank order."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return stats_u8
    out = torch.empty(world * stats_u8.numel(), dtype=torch.uint8, device=stats_u8.device)
    dist.all_gather_into_tensor(out, stats_u8)
    return out


def max_over_ranks(value: float, device) -> float:
    """Device-timed step time: the job's time is the slowest rank's."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t[0])


def sum_over_ranks(value: float, device) -> float:
    import torch
    import torch.distributed as dist
    t = torch.tensor([value], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t[0])


def stats_view(stats_u8) -> np.ndarray:
    """rs_replay_stats records as a numpy structured array."""
    return np.frombuffer(stats_u8.cpu().numpy().tobytes(), dtype=abi.STATS_DTYPE)

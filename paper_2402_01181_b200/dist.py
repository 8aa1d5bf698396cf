"""Multi-GPU plumbing (host side): one process per GPU over torch.distributed.

The hot path shards by independent units (environments / replica scenes), so
the data path has no collective; the only cross-rank traffic is the timing
reduction of the benchmark (max over ranks, BASELINE/bench contract) and the
optional gather of per-environment observations.
"""

from __future__ import annotations

import os


def world() -> tuple[int, int, int]:
    """(world_size, rank, local_rank) from the torchrun environment."""
    return (int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("RANK", "0")),
            int(os.environ.get("LOCAL_RANK", "0")))


def max_over_ranks(value: float, device=None) -> float:
    """Slowest rank's value (timings are reported as the max over ranks)."""
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(value: float, device=None) -> float:
    import torch
    import torch.distributed as dist

    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def throughput(units_local: float, seconds_local: float, device=None) -> float:
    """Whole-job throughput: units summed over ranks / slowest rank's time."""
    return sum_over_ranks(units_local, device) / max_over_ranks(seconds_local, device)

"""Multi-GPU sharding of independent traces (N4) — host-side logic, one process per GPU.

Units are independent (every (trace, grid, policy) is its own simulate() run), so
ranks own contiguous trace ranges and exchange nothing while computing. The single collective
reduces the int64 union-bin histogram (the global config histogram) — NCCL over NVLink on
B200, gloo in the CPU tests. Integer sums make the result independent of the rank count.
"""

from __future__ import annotations


def shard_range(n_traces: int, rank: int, world: int) -> tuple[int, int]:
    """[lo, hi) of the global trace ids owned by ``rank`` (contiguous, sizes differ by <= 1)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank/world {rank}/{world}")
    return n_traces * rank // world, n_traces * (rank + 1) // world


def reduce_histogram(hist, group=None):
    """Sum the per-rank union-bin histograms in place (int64; exact, order-independent)."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(hist, op=dist.ReduceOp.SUM, group=group)
    return hist


def max_over_ranks(value: float, device=None, group=None) -> float:
    """Device-timed durations are reported as the max over ranks."""
    import torch
    import torch.distributed as dist

    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t[0])

"""Element-range sharding across the GPUs of one node.

Elements are independent (integrate_generic has no cross-element term,
integrate_ref.cpp:50-91), so GPU g of G owns the contiguous range
[floor(g*E/G), floor((g+1)*E/G)) -- the multi-GPU analogue of the reference's
disjoint work-group ranges (kernels.cpp:98-100).  No collective touches the
data path; the only collectives are the barrier around the timed region and
the max-over-ranks reduction of device times.
"""
from __future__ import annotations


def rank_range(n_total: int, world: int, rank: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous share of n_total elements."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    lo = rank * n_total // world
    hi = (rank + 1) * n_total // world
    return lo, hi - lo


def max_over_ranks(value: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar (device times are reported as the slowest rank)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return float(value)
    import torch

    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())

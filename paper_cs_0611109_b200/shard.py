"""Stripe sharding across ranks.  Stripes are independent (each touches only
its own N+2 strips, Eq. (znparity)), so the data path needs no collective:
each rank processes its own stripes, and torch.distributed (NCCL on GPUs, gloo on CPU) is used
only to align the start of timing and to reduce times (max) and verification counters (sum).
"""
from __future__ import annotations


def block_range(rank: int, world: int, total: int) -> tuple[int, int]:
    """Contiguous block partition of `total` stripes: rank r gets [floor(r*S/G), floor((r+1)*S/G))."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad rank/world/total")
    return (rank * total) // world, ((rank + 1) * total) // world


def weak_range(rank: int, per_rank: int) -> tuple[int, int]:
    """Weak scaling: every rank owns `per_rank` stripes with distinct global indices."""
    return rank * per_rank, (rank + 1) * per_rank


def max_over_ranks(value: float, device=None) -> float:
    """Max of a per-rank scalar (e.g. elapsed ms) over the default process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _coll_device(device):
    """NCCL reduces device tensors; gloo (CPU tests, 1-GPU rehearsal) reduces host tensors."""
    import torch.distributed as dist
    return device if dist.get_backend() == "nccl" else "cpu"


def sum_over_ranks(values, device=None) -> list[int]:
    """Elementwise sum of per-rank integer counters over the default process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [int(v) for v in values]
    t = torch.tensor([int(v) for v in values], dtype=torch.int64, device=_coll_device(device))
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [int(v) for v in t.tolist()]


def gather_over_ranks(value: float, device=None) -> list[float]:
    """Per-rank values of a scalar (e.g. each rank's elapsed ms), in rank order."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return [float(value)]
    dev = _coll_device(device)
    t = torch.tensor([float(value)], dtype=torch.float64, device=dev)
    out = [torch.zeros_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(out, t)
    return [float(x.item()) for x in out]

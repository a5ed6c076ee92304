"""Multi-GPU sharding of env ranges and the rollout-statistics all-reduce.

Environments are independent, so a batch shards by contiguous
global env ranges with no data-path collective: rank r owns
[offset_r, offset_r + n_r) and keys its Philox streams by the GLOBAL index,
which makes every trajectory independent of the GPU count (the reference's
worker-invariance contract, engine.py:471-484).  The only collective is one
all-reduce of ~8 float64 rollout statistics (NCCL over NVLink/NVSwitch on
the GPU box, gloo in the CPU tests).
"""

from __future__ import annotations

import torch


def shard_range(n_global: int, rank: int, world: int) -> tuple:
    """(offset, count) of rank's contiguous slice; same split as np.linspace bounds."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    lo = (n_global * rank) // world
    hi = (n_global * (rank + 1)) // world
    return lo, hi - lo


def dist_ready(group=None) -> bool:
    return torch.distributed.is_available() and torch.distributed.is_initialized()


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """Sum ``t`` over the process group in place (no-op when not distributed)."""
    if dist_ready(group):
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.SUM, group=group)
    return t


def allreduce_max(x: float, device, group=None) -> float:
    """Max of a host scalar over ranks (used for device-timed max-over-ranks)."""
    if not dist_ready(group):
        return x
    t = torch.tensor([x], dtype=torch.float64, device=device)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX, group=group)
    return float(t.item())

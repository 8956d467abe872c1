"""Multi-GPU plumbing: independent environment+query units
are sharded across ranks with no data-path collective; the only exchange is
one all-gather of the fixed-size 48-byte result records (mpap_result) per
batch, never inside the wave loop.  torch.distributed with NCCL on GPUs
(gloo on CPU for tests).
"""
from __future__ import annotations

from typing import List

import numpy as np


def shard_envs(rank: int, world: int, per_rank: int) -> List[int]:
    """Weak scaling: rank r owns env indices [r*Q, (r+1)*Q)."""
    if not (0 <= rank < world) or per_rank < 0:
        raise ValueError("bad rank/world/per_rank")
    return list(range(rank * per_rank, (rank + 1) * per_rank))


def gather_results(local, world: int):
    """All-gather a uint8 tensor of result records (equal size on every rank)
    into one tensor ordered by rank."""
    import torch
    import torch.distributed as dist
    if world == 1:
        return local
    if dist.get_backend() == "nccl":
        out = torch.empty(world * local.numel(), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, local)
        return out
    parts = [torch.empty_like(local) for _ in range(world)]
    dist.all_gather(parts, local)
    return torch.cat(parts)


def records(tensor, dtype) -> np.ndarray:
    """View gathered bytes as structured result records."""
    return tensor.cpu().numpy().view(dtype)


def mc_trial_shard(rank: int, world: int, trials: int):
    """Monte Carlo trials of one plan split across ranks (NEXT-4: trials are
    independent counter-based streams, so rank r runs trials [t0, t0 + n) and
    the per-trial results equal a single-GPU run's).  Returns (t0, n)."""
    if not (0 <= rank < world) or trials < 0:
        raise ValueError("bad rank/world/trials")
    base, extra = divmod(trials, world)
    t0 = rank * base + min(rank, extra)
    return t0, base + (1 if rank < extra else 0)


def reduce_exceed(local):
    """Sum the per-plan exceedance counts (int64 tensor) over ranks: the one
    collective of a sharded Monte Carlo verification."""
    import torch.distributed as dist
    if dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(local, op=dist.ReduceOp.SUM)
    return local

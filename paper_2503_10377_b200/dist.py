"""Head sharding over the GPUs of one node.

Heads are independent in attention, so rank g of G owns heads
[g*h/G, (g+1)*h/G) — the post-all-to-all layout of Ulysses-style sequence
parallelism (P:575, P:594 [§7.3, §8]) without the all-to-all, because inputs are
generated head-sharded.  There is no collective inside a step; the only
collectives are the timing reduction (max over ranks) and one all-gather of the
results after timing (NCCL over NVLink on GPUs, gloo on CPU in tests).
"""

from __future__ import annotations

import torch


def head_range(heads: int, world: int, rank: int):
    """Global head indices owned by ``rank``."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    if heads % world:
        raise ValueError(f"heads={heads} not divisible by {world} ranks")
    per = heads // world
    return list(range(rank * per, (rank + 1) * per))


def max_over_ranks(x: float, world: int, device=None) -> float:
    """Max of a per-rank scalar (the step time) over all ranks."""
    if world == 1:
        return float(x)
    import torch.distributed as dist
    if dist.get_backend() != "nccl":
        device = "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_heads(local: torch.Tensor, world: int) -> torch.Tensor:
    """All-gather a head-sharded token-major tensor [S, h/G, d] into [S, h, d]
    (rank order = head order)."""
    if world == 1:
        return local
    import torch.distributed as dist
    local = local.contiguous()
    if dist.get_backend() != "nccl":  # gloo (CPU tests): gather host copies
        local = local.cpu()
    parts = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    if local.is_cuda:
        dist.all_gather_into_tensor(parts, local)  # NCCL over NVLink / NVSwitch
    else:
        dist.all_gather(list(parts.unbind(0)), local)
    # [G, S, h/G, d] -> [S, G*h/G, d]
    return parts.permute(1, 0, 2, 3).reshape(local.shape[0], world * local.shape[1], local.shape[2])

"""Direction sharding across ranks.

CSFD perturbation directions are independent full-pipeline evaluations whose
real channel is identical, so rank r of N packs a contiguous
block of the direction list as its channels and recomputes the shared real
pipeline; there is no per-frame exchange.  The only collective is the final
gather of the derivative columns (C2).  `gather_columns` uses
torch.distributed (NCCL on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

from typing import List, Sequence, Tuple


def shard_directions(dirs: Sequence[int], world: int, rank: int) -> Tuple[int, List[int]]:
    """Contiguous block of `dirs` owned by `rank`: (offset, directions).  Block
    sizes differ by at most one (the first len(dirs) % world ranks get one
    more)."""
    if world <= 0 or not (0 <= rank < world):
        raise ValueError("bad world/rank")
    n = len(dirs)
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    size = base + (1 if rank < extra else 0)
    return start, list(dirs[start:start + size])


def gather_columns(local_grad, n_total: int, world: int, rank: int, group=None):
    """All-gather every rank's derivative columns into the full gradient
    (float64, length n_total) on every rank."""
    import torch
    import torch.distributed as dist

    dev = local_grad.device
    sizes = [shard_directions(range(n_total), world, r)[1].__len__() for r in range(world)]
    width = max(sizes) if sizes else 0
    buf = torch.zeros(width, dtype=torch.float64, device=dev)
    buf[: local_grad.numel()] = local_grad.to(torch.float64)
    out = [torch.zeros(width, dtype=torch.float64, device=dev) for _ in range(world)]
    dist.all_gather(out, buf, group=group)
    return torch.cat([out[r][: sizes[r]] for r in range(world)])

"""Direction sharding across ranks.

CSFD perturbation directions are independent full-pipeline evaluations whose
real channel is identical, so rank r of N packs a contiguous
block of the direction list as its channels and recomputes the shared real
pipeline; there is no per-frame exchange.  The only collective is the final
gather of the derivative columns (C2): `gather_columns_native` runs it in the
C-ABI (csf_gather_columns over the context's NCCL communicator);
`gather_columns` is the torch.distributed form (gloo in the CPU tests).
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


def attach_native_comm(ctx, world: int, rank: int) -> None:
    """Give the context its NCCL communicator: rank 0 creates the unique id,
    torch.distributed (already initialised) broadcasts it."""
    import torch.distributed as dist
    import paper_2405_02187_b200 as csf
    obj = [csf.comm_unique_id() if rank == 0 else None]
    if world > 1:
        dist.broadcast_object_list(obj, src=0)
    ctx.attach_comm(world, rank, obj[0])


def gather_columns_native(ctx, local_grad, n_total: int, world: int):
    """All-gather every rank's derivative columns through csf_gather_columns."""
    counts = [len(shard_directions(range(n_total), world, r)[1]) for r in range(world)]
    return ctx.gather_columns(local_grad, counts)

"""Pair sharding across ranks: independent scan pairs split by
pair index into contiguous blocks, no collective on the hot path; only the
per-pair results are gathered to rank 0 afterwards."""
from __future__ import annotations


def shard_range(total: int, world: int, rank: int) -> tuple[int, int]:
    """(first, count) of rank's contiguous block; the first total % world ranks get one extra."""
    if world < 1 or not (0 <= rank < world) or total < 0:
        raise ValueError("bad shard arguments")
    base, extra = divmod(total, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def gather_results(local, total: int, world: int, rank: int, group=None):
    """Gather each rank's result rows (torch tensor [count, ...]) into a [total, ...]
    tensor on rank 0 in pair order. Returns None on the other ranks."""
    import torch
    import torch.distributed as dist

    if world == 1:
        return local
    if dist.get_backend(group) == "gloo":  # gloo gathers host tensors only
        local = local.cpu()
    counts = [shard_range(total, world, r)[1] for r in range(world)]
    width = max(counts)
    pad = torch.zeros((width,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == 0 else None
    dist.gather(pad, bufs, dst=0, group=group)
    if rank != 0:
        return None
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)

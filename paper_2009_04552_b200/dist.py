"""Host-side plumbing of the multi-GPU path:
contiguous row ranges (north_star: "points are partitioned into contiguous
ranges"), the NCCL unique-id broadcast over torch.distributed, and the
max-over-ranks timing reduction.  No arithmetic of the method lives here: every
collective the method needs (core-bit OR, per-round MIN of the packed keys) is
issued by libkdb.so itself on its own NCCL communicator.
"""
from __future__ import annotations


def rank_rows(n_total: int, rank: int, world: int) -> tuple[int, int]:
    """Rows [floor(r N / P), floor((r+1) N / P)) of rank r -- the same split the
    library's sim communicator uses for its virtual ranks."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return n_total * rank // world, n_total * (rank + 1) // world


def share_nccl_id(rank: int, make_id, group=None) -> bytes:
    """Rank 0 creates the 128-byte ncclUniqueId (``make_id()``) and every rank
    receives the same bytes through torch.distributed (any backend)."""
    import torch.distributed as dist
    obj = [make_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    uid = obj[0]
    if not isinstance(uid, (bytes, bytearray)) or len(uid) != 128:
        raise RuntimeError("bad NCCL unique id")
    return bytes(uid)


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The max of a per-rank time over all ranks (bench.py: a step lasts as long
    as its slowest rank)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


def gather_rows(col, group=None):
    """Concatenate every rank's 1-D tensor ``col`` (this rank's rows of a
    per-row quantity, any length) in rank order on every rank: the eps rule's
    median is over ALL rows (bench.py builds only its own rows of the graph)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size(group) == 1:
        return col
    world = dist.get_world_size(group)
    n = torch.tensor([col.numel()], dtype=torch.int64, device=col.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    mx = int(max(int(x.item()) for x in sizes))
    pad = torch.zeros(mx, dtype=col.dtype, device=col.device)
    pad[:col.numel()] = col
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:int(k.item())] for p, k in zip(parts, sizes)])

"""Rank bookkeeping for SPMD launches (one process per GPU, torch.distributed).

The row/CN partition follows include/pnn.h: rank r of G owns CNs
[floor(r·K/G), floor((r+1)·K/G)) and exactly the rows of their slices
(PAPER.md:166-169 slicing, reading R17), so no training data moves between
GPUs and the only exchange is the merge's all-reduce.
"""
from __future__ import annotations


def slice_bounds(N: int, K: int, i: int):
    """R17: CN i of K gets rows [start, start + count), count = floor(N/K) + [i < N mod K]."""
    base, rem = divmod(N, K)
    return i * base + min(i, rem), base + (1 if i < rem else 0)


def rank_subnets(K: int, world: int, rank: int):
    """CNs [first, first + count) owned by `rank`."""
    first = rank * K // world
    return first, (rank + 1) * K // world - first


def rank_rows(N: int, K: int, world: int, rank: int):
    """Rows [start, start + count) this rank trains on: its CNs' slices, concatenated."""
    first, cnt = rank_subnets(K, world, rank)
    if cnt == 0:      # K < G: an idle rank (contributes zeros to the merge)
        return (slice_bounds(N, K, first)[0] if first < K else N), 0
    s0, _ = slice_bounds(N, K, first)
    s1, c1 = slice_bounds(N, K, first + cnt - 1)
    return s0, s1 + c1 - s0


def nccl_unique_id_bytes(rank: int, group=None) -> bytes:
    """Create an ncclUniqueId on rank 0 (via torch's NCCL bindings) and broadcast it
    with torch.distributed (no process group: a single process, the id as made);
    returns the 128 raw bytes on every rank."""
    import torch
    import torch.distributed as dist
    if rank == 0:
        uid = bytes(torch.cuda.nccl.unique_id())
    else:
        uid = bytes(128)
    if not dist.is_initialized():
        return uid
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]

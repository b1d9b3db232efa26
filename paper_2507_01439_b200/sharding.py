"""Pair-level data parallelism over ranks.

Registration pairs are independent, so the path shards at pair granularity with no data-path collective:
rank r of G takes the contiguous pair range [floor(r·P/G), floor((r+1)·P/G)).  The only exchange is the
gather of fixed-size result records (104 B each, padded to ceil(P/G) per rank) with one
``all_gather_into_tensor`` — NCCL over NVLink on GPUs, gloo in the CPU tests — after which every rank
holds all results in global pair order.
"""
from __future__ import annotations

import numpy as np

from ._binding import RESULT_DTYPE


def shard_range(num_pairs: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous [begin, end) pair range of `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world or num_pairs < 0:
        raise ValueError("bad shard arguments")
    return (rank * num_pairs) // world, ((rank + 1) * num_pairs) // world


def gather_results(local, num_pairs: int, group=None):
    """All-gather per-pair result records (numpy RESULT_DTYPE array, or a uint8 tensor of records) from every
    rank of `group`; returns a numpy RESULT_DTYPE array of length num_pairs in global pair order."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    cap = -(-num_pairs // world)  # ceil
    isz = RESULT_DTYPE.itemsize
    if isinstance(local, np.ndarray):
        raw = torch.from_numpy(np.ascontiguousarray(local).view(np.uint8).copy())
    else:
        raw = local.reshape(-1)
    backend = dist.get_backend(group)
    device = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(cap * isz, dtype=torch.uint8, device=device)
    buf[: raw.numel()] = raw.to(device)
    out = torch.empty(world * cap * isz, dtype=torch.uint8, device=device)
    dist.all_gather_into_tensor(out, buf, group=group)
    full = out.cpu().numpy().reshape(world, cap * isz)
    parts = []
    for r in range(world):
        b, e = shard_range(num_pairs, world, r)
        parts.append(full[r, : (e - b) * isz])
    del rank
    return np.concatenate(parts).view(RESULT_DTYPE)

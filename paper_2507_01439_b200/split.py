"""NEXT(1): one registration pair split over several GPUs.

The paper's "Pivot-level Parallelism" carried across ranks for large N: every
rank runs the library's split phases (include/turboreg.h "NEXT(1)") on the same pair and the ranks exchange
three buffers in between:

  phase 1  turboreg_split_begin   compat on this rank's block-row pairs      -> all_reduce(SUM) of C's words
  phase 2  turboreg_split_sc2     SC^2 assembly of this rank's work items     -> all_reduce(SUM) of E edge words
  phase 3  turboreg_split_search  PGS / Kabsch / scoring of its pivot slice   -> all_gather of 104-byte records
  phase 4  turboreg_split_merge   T* = argmax of the gathered records (on the GPU)

Every word of C and every O2 edge word is written by exactly one rank into a zeroed buffer, so SUM rebuilds
the full arrays; pivot selection then runs on identical data on every rank.  Bytes on NVLink per rank (ring
all-reduce, G ranks): 2(G-1)/G x (N²/8 + 4E) + G x 104 — at N = 32768, E ≈ 2.4e7: ≈ 0.23 + 0.18 GB.

This module only sequences calls and collectives (torch.distributed: NCCL on GPUs); every step of the path
runs in libturboreg.so.  `engine` is a TurboReg context or any object with the same split_* methods (the
CPU gloo tests use a stand-in).
"""
from __future__ import annotations

from ._binding import RESULT_DTYPE, SPLIT_BITS, SPLIT_EDGES, SPLIT_RESULT


def register_split(engine, src, dst, group=None, stream=None):
    """Register one pair over the ranks of `group` (each rank calls this with the same pair); returns the
    result dict of turboreg_register on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    st = engine.split_begin(src, dst, rank, world, stream)
    if st != 0:  # n out of range: the same on every rank, nothing to exchange
        return {"status": st}
    bits = engine.split_tensor(SPLIT_BITS)
    with _on(stream):
        dist.all_reduce(bits, op=dist.ReduceOp.SUM, group=group)
    e = engine.split_sc2(stream)
    if e > 0:
        edges = engine.split_tensor(SPLIT_EDGES, e)
        with _on(stream):
            dist.all_reduce(edges, op=dist.ReduceOp.SUM, group=group)
    engine.split_search(stream)
    part = engine.split_tensor(SPLIT_RESULT)
    parts = torch.empty(world * RESULT_DTYPE.itemsize, dtype=torch.uint8, device=part.device)
    with _on(stream):
        dist.all_gather_into_tensor(parts, part, group=group)
    return engine.split_merge(parts, world, stream)


def emulate_split(engines, src, dst):
    """The same phases and exchanges for G logical ranks on ONE device (engines[r] = rank r's context, run
    one after another; the collectives become sums / concatenations of their buffers).  For tests: the
    kernels of different ranks never wait on each other."""
    import torch

    g = len(engines)
    st = [e.split_begin(src, dst, r, g) for r, e in enumerate(engines)]
    if st[0] != 0:
        return {"status": st[0]}
    _sum_into([e.split_tensor(SPLIT_BITS) for e in engines])
    es = [e.split_sc2() for e in engines]
    assert len(set(es)) == 1, es
    if es[0] > 0:
        _sum_into([e.split_tensor(SPLIT_EDGES, es[0]) for e in engines])
    for e in engines:
        e.split_search()
    parts = torch.cat([e.split_tensor(SPLIT_RESULT) for e in engines])
    return engines[0].split_merge(parts, g)


def _sum_into(bufs):
    torch = _torch()
    with torch.cuda.device(bufs[0].device):
        torch.cuda.synchronize()
        total = bufs[0].clone()
        for b in bufs[1:]:
            total += b
        for b in bufs:
            b.copy_(total)
        torch.cuda.synchronize()


def _torch():
    import torch

    return torch


class _on:
    """`with torch.cuda.stream(s)` when s is a torch stream, else a no-op (the current stream)."""

    def __init__(self, stream):
        self.s = stream

    def __enter__(self):
        torch = _torch()
        self.cm = torch.cuda.stream(self.s) if isinstance(self.s, torch.cuda.Stream) else None
        if self.cm:
            self.cm.__enter__()

    def __exit__(self, *a):
        if self.cm:
            self.cm.__exit__(*a)

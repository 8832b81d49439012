"""Multi-GPU plumbing for the walk engine: one process per GPU.

Walks are independent and their streams are keyed by the walk id, so the
path shards with no data-path collective: rank r of W takes a contiguous
walk range (the reference's per-thread chunking, engine.cpp:437-455), and
the per-terminal tallies (sum, sum of squares, landed count) are combined
once with an all-reduce (NCCL over NVLink on GPUs, gloo in the CPU tests).
"""
from __future__ import annotations

import math

import numpy as np


def rank_range(total: int, rank: int, world: int) -> tuple[int, int]:
    """[begin, end) of this rank's walks: contiguous chunks, the first
    total % world ranks one longer (engine.cpp:440-455)."""
    chunk, extra = divmod(total, world)
    begin = rank * chunk + min(rank, extra)
    return begin, begin + chunk + (1 if rank < extra else 0)


def combine_tallies(sum_, sumsq, landed, device=None):
    """All-reduce per-terminal tallies over the default process group."""
    import torch
    import torch.distributed as dist
    t = torch.tensor(np.concatenate([np.asarray(sum_, np.float64), np.asarray(sumsq, np.float64)]),
                     dtype=torch.float64, device=device)
    n = torch.tensor(np.asarray(landed, np.int64), dtype=torch.int64, device=device)
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t)
        dist.all_reduce(n)
    k = len(sum_)
    tc = t.cpu().numpy()
    return tc[:k], tc[k:], n.cpu().numpy().astype(np.uint64)


def estimates(sum_, sumsq, walks):
    """Mean and standard error per slot, engine.cpp:388-400."""
    w = float(walks)
    out = []
    for s1, s2 in zip(sum_, sumsq):
        mean = s1 / w
        se = 0.0
        if walks > 1:
            se = math.sqrt(max(0.0, (s2 - s1 * s1 / w) / (w - 1)) / w)
        out.append((mean, se))
    return out

"""Sample sharding across GPUs.

Every token's computation is a pure function of its own sample's prefix
(model.hpp:54-57) and outputs are invariant to batch composition
(test_engine.cpp:307-320), so samples shard across ranks with no collective in
the verify step; weights are replicated.  Global sample ids are kept so the
synthetic prompts / seeds of a sample do not depend on the rank count.  The
only collective is the end-of-run gather of the per-sample outputs.
"""
from __future__ import annotations

import numpy as np


def local_ids(batch_per_rank: int, rank: int) -> list[int]:
    """Weak scaling: rank r owns global samples [r*B, (r+1)*B)."""
    return list(range(rank * batch_per_rank, (rank + 1) * batch_per_rank))


def split_ids(global_batch: int, world: int, rank: int) -> list[int]:
    """Strong scaling: contiguous, balanced blocks of a fixed global batch."""
    base, extra = divmod(global_batch, world)
    start = rank * base + min(rank, extra)
    return list(range(start, start + base + (1 if rank < extra else 0)))


def split_ids_by_length(prompt_lens: list[int], world: int, rank: int) -> list[int]:
    """Strong scaling balanced by prompt length: contiguous
    blocks (rank order stays global sample order, so the end-of-run gather
    needs no permutation) whose prompt-token totals are as even as the
    boundaries allow -- rank r's block ends where the prefix sum first reaches
    (r + 1) / world of the total, and every rank keeps at least one sample
    while there are enough."""
    n = len(prompt_lens)
    cum = np.cumsum(np.asarray(prompt_lens, dtype=np.int64))
    total = int(cum[-1]) if n else 0
    bounds = [0]
    for r in range(1, world):
        target = total * r / world
        b = int(np.searchsorted(cum, target, side="left")) + 1  # first prefix reaching the target
        b = max(b, bounds[-1] + (1 if n - bounds[-1] > world - r else 0))
        b = min(b, n - (world - r) if n >= world else n)
        bounds.append(max(b, bounds[-1]))
    bounds.append(n)
    return list(range(bounds[rank], bounds[rank + 1]))


def pad_tokens(seqs: list[list[int]], width: int) -> np.ndarray:
    out = np.full((len(seqs), width), -1, dtype=np.int32)
    for i, s in enumerate(seqs):
        out[i, : len(s)] = s
    return out


def gather_outputs(seqs: list[list[int]], width: int, dist, device=None) -> list[list[int]]:
    """all_gather the per-sample token streams of every rank (rank order =
    global sample order for contiguous shards).  `dist` is torch.distributed
    (NCCL on GPUs, gloo in the CPU tests)."""
    import torch

    t = torch.from_numpy(pad_tokens(seqs, width))
    if device is not None:
        t = t.to(device)
    n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
    sizes = [torch.zeros_like(n) for _ in range(dist.get_world_size())]
    dist.all_gather(sizes, n)
    mx = int(max(s.item() for s in sizes))
    if t.shape[0] < mx:
        t = torch.cat([t, torch.full((mx - t.shape[0], width), -1, dtype=t.dtype, device=t.device)])
    parts = [torch.empty_like(t) for _ in range(dist.get_world_size())]
    dist.all_gather(parts, t)
    out = []
    for s, p in zip(sizes, parts):
        for row in p[: int(s.item())].cpu().numpy():
            out.append([int(x) for x in row if x >= 0])
    return out

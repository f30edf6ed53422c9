"""Multi-GPU: equal-work contiguous shards of the linear edge range, one rank
per GPU, and the only collective on the path -- a final reduce of the summary
statistics.  Edge payload bytes never move between GPUs: shard g
is exactly bytes [bounds[g], bounds[g+1]) of the payload, so concatenating the
shards in rank order is the payload.

The reference's counterpart is the fork pool over contiguous chunks
(engine.py:262-276); partition invariance (tests/test_engine.py:92-101) is what
makes sharding a pure scheduling choice.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Optional

import numpy as np


def equal_work_bounds(lengths, parts: int) -> np.ndarray:
    """Host arithmetic identical to nwap_equal_work_bounds (csrc/nwap.cu): split
    [0, P) into ``parts`` contiguous ranges with (near) equal sum of len_r*len_c.
    bounds[g] = smallest linear index whose exclusive prefix work >= ceil(g*W/parts)."""
    L = np.asarray(lengths, dtype=np.int64)
    n = int(L.size)
    if n < 2 or parts < 1:
        raise ValueError("need n >= 2 and parts >= 1")
    P = n * (n - 1) // 2
    pre = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(L, out=pre[1:])
    roww = L * (pre[n] - pre[1:])
    rowpref = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(roww, out=rowpref[1:])
    W = int(rowpref[n])
    bounds = np.zeros(parts + 1, dtype=np.int64)
    for g in range(1, parts):
        target = (W * g + parts - 1) // parts
        r = int(np.searchsorted(rowpref[1:], target, side="left"))
        r = min(r, n - 2)
        need = target - int(rowpref[r])
        col = r + 1
        if need > 0:
            lr = int(L[r])
            k = (need + lr - 1) // lr
            col = int(np.searchsorted(pre, int(pre[r + 1]) + k, side="left"))
        idx = r * (2 * n - r - 1) // 2 + (col - r - 1)
        bounds[g] = min(max(idx, int(bounds[g - 1])), P)
    bounds[parts] = P
    return bounds


def shard_of(bounds: np.ndarray, rank: int):
    return int(bounds[rank]), int(bounds[rank + 1])


@dataclass
class ShardStats:
    sum: int
    count: int
    min: int
    max: int
    hist: Optional[np.ndarray] = None      # int64[256]
    degree: Optional[np.ndarray] = None    # int64[n]


def reduce_stats(local: ShardStats, group=None, device=None) -> ShardStats:
    """All-reduce per-shard statistics: SUM for sum/count/hist/degree, MIN/MAX for
    the extrema.  Works on any initialised torch.distributed backend (NCCL with
    CUDA tensors on the GPU box, gloo with CPU tensors in the CPU tests)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
            else torch.device("cpu")
    parts = [torch.tensor([local.sum, local.count], dtype=torch.int64)]
    has_hist = local.hist is not None
    has_deg = local.degree is not None
    if has_hist:
        parts.append(torch.as_tensor(np.asarray(local.hist, dtype=np.int64)))
    if has_deg:
        parts.append(torch.as_tensor(np.asarray(local.degree, dtype=np.int64)))
    sums = torch.cat(parts).to(device)
    ext = torch.tensor([local.min, -local.max], dtype=torch.int64, device=device)
    dist.all_reduce(sums, op=dist.ReduceOp.SUM, group=group)
    dist.all_reduce(ext, op=dist.ReduceOp.MIN, group=group)
    sums = sums.cpu().numpy()
    ext = ext.cpu().numpy()
    pos = 2
    hist = degree = None
    if has_hist:
        hist = sums[pos:pos + 256].copy()
        pos += 256
    if has_deg:
        degree = sums[pos:].copy()
    return ShardStats(int(sums[0]), int(sums[1]), int(ext[0]), int(-ext[1]), hist, degree)


def gather_counts(local_count: int, group=None, device=None):
    """All-gather of per-shard kept-edge counts (placement of compacted lists)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return [int(local_count)]
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" \
            else torch.device("cpu")
    mine = torch.tensor([local_count], dtype=torch.int64, device=device)
    out = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, mine, group=group)
    return [int(t.item()) for t in out]

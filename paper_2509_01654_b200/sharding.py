"""Multi-GPU: equal-work contiguous shards of the linear edge range, one rank
per GPU, and the only collective on the path -- a final reduce of the summary
statistics and degree counts plus a gather of the kept-edge counts.
Edge payload bytes never move between GPUs: shard g is exactly bytes
[bounds[g], bounds[g+1]) of the payload, so concatenating the shards in rank order
is the payload, and concatenating the per-shard kept lists in rank order is the
kept list of the whole job.

The reference's counterpart is the fork pool over contiguous chunks
(engine.py:262-276); partition invariance (tests/test_engine.py:92-101) is what
makes sharding a pure scheduling choice.

``run_shard`` is the rank-level driver: bounds -> score my shard on my GPU ->
(optional) threshold compaction + degree -> all-reduce -> all-gather.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import List, Optional, Tuple

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

    @property
    def mean(self) -> float:
        return self.sum / self.count if self.count else float("nan")


def _collective_device(group, device):
    import torch
    import torch.distributed as dist

    if device is not None:
        return torch.device(device)
    if dist.get_backend(group) == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def reduce_stats(local: ShardStats, group=None, device=None) -> ShardStats:
    """All-reduce per-shard statistics: SUM for sum/count/hist/degree, MIN/MAX for
    the extrema.  Works on any initialised torch.distributed backend (NCCL with
    CUDA tensors on the GPU box, gloo with CPU tensors in the CPU tests).  ``hist`` and
    ``degree`` may be numpy arrays or torch tensors (a CUDA degree tensor is reduced in
    place over NCCL without a host round trip)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return local
    device = _collective_device(group, device)

    def as_i64(x):
        t = x if isinstance(x, torch.Tensor) else torch.as_tensor(np.asarray(x, dtype=np.int64))
        return t.to(device=device, dtype=torch.int64)

    parts = [torch.tensor([local.sum, local.count], dtype=torch.int64, device=device)]
    has_hist = local.hist is not None
    has_deg = local.degree is not None
    if has_hist:
        parts.append(as_i64(local.hist))
    if has_deg:
        parts.append(as_i64(local.degree))
    sums = torch.cat(parts)
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
    device = _collective_device(group, device)
    mine = torch.tensor([local_count], dtype=torch.int64, device=device)
    out = [torch.zeros_like(mine) for _ in range(dist.get_world_size(group))]
    dist.all_gather(out, mine, group=group)
    return [int(t.item()) for t in out]


@dataclass
class ShardResult:
    """What one rank holds after ``run_shard``."""

    rank: int
    world: int
    start: int                      # this rank's linear edge range [start, end)
    end: int
    payload: object = None          # int8 device tensor of end-start scores (dense mode, passes == 1), else None
    local: ShardStats = None        # this shard's statistics
    total: ShardStats = None        # all shards reduced: sum/count/min/max (+ hist, + degree of the whole graph)
    kept_idx: object = None         # int64 device tensor: kept edges of this shard, increasing index
    kept_score: object = None       # int8 device tensor
    kept_counts: List[int] = field(default_factory=list)    # kept edges per rank (all-gather)
    kept_offset: int = 0            # position of this shard's kept list in the whole job's kept list
    bounds: Optional[np.ndarray] = None


def run_shard(ctx, rank: int, world: int, *, threshold: Optional[int] = None,
              normalized: Optional[Tuple[float, float]] = None, dense: bool = True, out=None, passes: int = 1,
              want_hist: bool = False, want_degree: Optional[bool] = None, capacity: Optional[int] = None,
              variant: str = "auto", group=None, collective_device=None) -> ShardResult:
    """Rank-level driver of the all-pairs job (the counterpart of one worker of the reference's pool,
    engine.py:262-276, plus the final accumulation of engine.py:246-260 as a collective).

    1. ``bounds = ctx.equal_work_bounds(world)``; this rank owns ``[bounds[rank], bounds[rank+1])``.
    2. Score the shard on this rank's GPU: ``dense=True`` into ``out`` (allocated when None; with
       ``passes > 1`` the shard is scored as that many equal-work sub-ranges into ONE reused buffer of the
       largest sub-range, for shards larger than HBM, and no payload is returned).
       With ``threshold`` / ``normalized`` the kept edges and (``want_degree``, default on) the degree
       counts are produced too: from the dense buffer by ``compact_range`` / ``filter_normalized``, or, with
       ``dense=False``, by the sparse-output kernel with no payload at all.
       ``want_hist`` adds the 256-bin raw histogram (``k_payload_stats`` over the dense buffer).
    3. ``reduce_stats`` of {sum, count, min, max, hist, degree} and ``gather_counts`` of the kept counts:
       the only communication of the whole job.
    """
    import torch

    if threshold is not None and normalized is not None:
        raise ValueError("pass at most one of threshold / normalized")
    filtering = threshold is not None or normalized is not None
    if not dense and not filtering:
        raise ValueError("dense=False needs a threshold or a normalised range: there would be no output")
    if want_hist and not dense:
        raise ValueError("the histogram is computed from the dense shard")
    if want_degree is None:
        want_degree = filtering
    bounds = np.asarray(ctx.equal_work_bounds(world), dtype=np.int64)
    s, e = shard_of(bounds, rank)
    dev = getattr(ctx, "torch_device", None) or torch.device("cuda", ctx.device)
    n = ctx.n
    passes = max(1, int(passes))
    if passes == 1:
        sub = [(s, e)]
    else:
        fine = np.asarray(ctx.equal_work_bounds(world * passes), dtype=np.int64)
        sub = [(int(fine[rank * passes + k]), int(fine[rank * passes + k + 1])) for k in range(passes)]
        assert sub[0][0] == s and sub[-1][1] == e
    degree = torch.zeros(n, dtype=torch.int32, device=dev) if (filtering and want_degree) else None
    if capacity is None:
        capacity = max(1 << 20, (e - s) // 1000)
    acc = [0, 127, -128, 0]
    hist = np.zeros(256, dtype=np.int64) if want_hist else None
    kept_i, kept_s = [], []

    def add(st):
        acc[0] += st[0]
        acc[1] = min(acc[1], st[1])
        acc[2] = max(acc[2], st[2])
        acc[3] += st[3]

    payload = None
    if dense:
        need = max(b - a for a, b in sub)
        if out is None:
            out = torch.empty(max(need, 1), dtype=torch.int8, device=dev)
        elif out.numel() < need:
            raise ValueError(f"out holds {out.numel()} bytes, the shard needs {need}")
        for a, b in sub:
            if b <= a:
                continue
            add(ctx.score_range(a, b, out, variant=variant)[:4])
            if want_hist:
                hist += ctx.payload_stats(out, b - a)[4]
            if threshold is not None:
                ki, ks = ctx.compact_range(out, a, b, threshold, capacity, degree=degree)
            elif normalized is not None:
                ki, ks = ctx.filter_normalized(out, a, b, normalized[0], normalized[1], capacity, degree=degree)
            if filtering:
                kept_i.append(ki.clone() if passes > 1 else ki)
                kept_s.append(ks.clone() if passes > 1 else ks)
        payload = out[: e - s] if passes == 1 else None
    else:
        for a, b in sub:
            if b <= a:
                continue
            ki, ks, st = ctx.score_range_compact(a, b, threshold=threshold, normalized=normalized, capacity=capacity,
                                                 degree=degree, variant=variant)
            add(st)
            kept_i.append(ki)
            kept_s.append(ks)
    local = ShardStats(acc[0], acc[3], acc[1], acc[2], hist, degree)
    total = reduce_stats(local, group=group, device=collective_device)
    if total is local and degree is not None:          # single process: same shape as the reduced result
        total = ShardStats(local.sum, local.count, local.min, local.max, hist, degree.to(torch.int64).cpu().numpy())
    res = ShardResult(rank=rank, world=world, start=s, end=e, payload=payload, local=local, total=total, bounds=bounds)
    if filtering:
        res.kept_idx = kept_i[0] if len(kept_i) == 1 else torch.cat(kept_i) if kept_i else torch.empty(0, dtype=torch.int64, device=dev)
        res.kept_score = kept_s[0] if len(kept_s) == 1 else torch.cat(kept_s) if kept_s else torch.empty(0, dtype=torch.int8, device=dev)
        res.kept_counts = gather_counts(int(res.kept_idx.numel()), group=group, device=collective_device)
        res.kept_offset = int(sum(res.kept_counts[:rank]))
    return res

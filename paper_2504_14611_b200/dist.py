"""Multi-GPU sharding of the hot path (one process per GPU, torch.distributed/NCCL).

The J-DOB instances are independent, so a batch shards into contiguous instance
ranges with no data-path collective; the only exchange is the statistics fold
(a12).  The brute-force index space shards into contiguous vector-aligned ranges
(each vector's j-scan stays on one rank); the exchange is a MIN-allreduce of
(E, idx) done as MIN over E followed by MIN over the indices of the ranks that hold
that E -- equal to the lowest-index tie-break of one sequential scan.

The functions take torch tensors on any device, so the same code runs over NCCL on
GPUs and over gloo on CPU (tests/test_dist_gloo.py).
"""
from __future__ import annotations

import contextlib
from typing import Tuple

STATS_MAX_FIELD, STATS_MIN_FIELD = 3, 4
IDX_NONE = 2 ** 62


def shard_range(n: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [begin, end) of n units for `rank` of `world` (sizes differ by <= 1)."""
    return n * rank // world, n * (rank + 1) // world


def bf_shard(size: int, k: int, world: int, rank: int) -> Tuple[int, int]:
    """Vector-aligned candidate range of `rank`: whole vectors (k grid points each)."""
    V = size // k
    v0, v1 = shard_range(V, world, rank)
    return v0 * k, v1 * k


def _nvtx(name):
    """NVTX range around a collective (SURVEY §5 tracing) when CUDA is present."""
    import torch
    if torch.cuda.is_available():
        return torch.cuda.nvtx.range(name)
    return contextlib.nullcontext()


def allreduce_stats(stats, dist):
    """Fold per-rank statistics [n_buckets, 80]: SUM, except field 3 MAX and field 4 MIN."""
    with _nvtx("jdob.allreduce_stats"):
        red = stats.clone()
        dist.all_reduce(red, op=dist.ReduceOp.SUM)
        mx = stats[:, STATS_MAX_FIELD].contiguous().clone()
        mn = stats[:, STATS_MIN_FIELD].contiguous().clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        red[:, STATS_MAX_FIELD] = mx
        red[:, STATS_MIN_FIELD] = mn
        return red


def fold_parts(parts):
    """Fold statistics roots [P, n_buckets, 80] (P a power of two, part order) pairwise -- the top of the
    dyadic tree of jdob_stats (include/jdob.h jdob_stats_part): fields add, except 3 (max) and 4 (min)."""
    import torch
    t = parts
    while t.shape[0] > 1:
        a, b = t[0::2], t[1::2]
        s = a + b
        s[:, :, STATS_MAX_FIELD] = torch.where(b[:, :, STATS_MAX_FIELD] > a[:, :, STATS_MAX_FIELD],
                                               b[:, :, STATS_MAX_FIELD], a[:, :, STATS_MAX_FIELD])
        s[:, :, STATS_MIN_FIELD] = torch.where(b[:, :, STATS_MIN_FIELD] < a[:, :, STATS_MIN_FIELD],
                                               b[:, :, STATS_MIN_FIELD], a[:, :, STATS_MIN_FIELD])
        t = s
    return t[0]


def fold_stats(stats, dist):
    """Global statistics from per-rank roots of jdob_stats_part (rank r = part r of world): all_gather
    of the [n_buckets, 80] roots (P x 40 KB at most) and the pairwise fold in rank order, on every rank.
    The same bits as one jdob_stats call over the whole batch when the world size is a power of two;
    otherwise the NCCL SUM/MAX/MIN fold (allreduce_stats), whose float sums are equal within 1e-9."""
    import torch
    world = dist.get_world_size()
    if world & (world - 1):
        return allreduce_stats(stats, dist)
    with _nvtx("jdob.fold_stats"):
        x = stats.contiguous()
        if dist.get_backend() == "gloo" and x.is_cuda:   # test-only backend: gather on the host
            x = x.cpu()
        parts = [torch.empty_like(x) for _ in range(world)]
        dist.all_gather(parts, x)
        return fold_parts(torch.stack(parts)).to(stats.device)


def allreduce_argmin(E, idx, dist):
    """Global (E, idx) lexicographic minimum of per-rank partial argmins (1-element tensors).

    idx < 0 (no feasible candidate on that rank) never wins unless every rank has none."""
    import torch
    with _nvtx("jdob.allreduce_argmin"):
        Eg = E.clone()
        dist.all_reduce(Eg, op=dist.ReduceOp.MIN)
        cand = torch.where((E == Eg) & (idx >= 0), idx, torch.full_like(idx, IDX_NONE))
        dist.all_reduce(cand, op=dist.ReduceOp.MIN)
        cand = torch.where(cand == IDX_NONE, torch.full_like(cand, -1), cand)
        return Eg, cand

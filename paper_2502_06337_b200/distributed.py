"""Sharded estimate_single over ranks (one process per GPU; torch.distributed is the plumbing).

SURVEY.md section 8(e): rank r owns the contiguous correspondence range
[N*r/P, N*(r+1)/P), preprocesses and votes it into a local uint32 grid; the grids are summed
with an all-reduce (NCCL over NVLink on B200; integer sums, so the result is bit-identical to the
single-GPU grid -- the reference's own chunked vote relies on the same property,
voting.cpp:102-117). The correspondences are all-gathered in rank order (reproducing input
order, hence the reference's kept/inlier index order) and every rank finishes the solve from the
reduced grid: identical estimate on all ranks, identical to the 1-GPU result.

The compute is behind a small backend interface so the same protocol runs on B200s
(`DeviceBackend`, the C-ABI) and, in the CPU test-suite, on the oracle over gloo.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank `rank`."""
    return n * rank // world, n * (rank + 1) // world


class DeviceBackend:
    """B200 backend: vote / finish through the C-ABI on the rank's GPU."""

    def __init__(self, ctx):
        self.ctx = ctx

    def vote_shard(self, shard: torch.Tensor, cfg) -> torch.Tensor:
        g = torch.empty((cfg.grid, cfg.grid), dtype=torch.int32, device=shard.device)  # uint32 bits
        self.ctx.vote_shard(shard.data_ptr(), shard.shape[0], g.data_ptr(), cfg)
        return g

    def finish(self, corrs: torch.Tensor, grid: torch.Tensor, cfg):
        return self.ctx.estimate_single_prevoted(corrs.data_ptr(), corrs.shape[0], grid.data_ptr(), cfg)


def all_gather_rows(shard: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """Rank-ordered concatenation of every rank's shard (shapes are known from shard_bounds)."""
    world = dist.get_world_size(group)
    sizes = [shard_bounds(n_total, world, r)[1] - shard_bounds(n_total, world, r)[0] for r in range(world)]
    width = max(sizes)
    padded = torch.zeros((width,) + tuple(shard.shape[1:]), dtype=shard.dtype, device=shard.device)
    padded[: shard.shape[0]] = shard
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)])


def sharded_estimate_single(shard: torch.Tensor, n_total: int, cfg, backend, group=None):
    """estimate_single over all ranks' shards; every rank returns the same estimate."""
    grid = backend.vote_shard(shard, cfg)
    dist.all_reduce(grid, op=dist.ReduceOp.SUM, group=group)  # int32 wrap-around == uint32 sum
    corrs = all_gather_rows(shard, n_total, group)
    return backend.finish(corrs, grid, cfg)


def batch_estimate(problems, cfg, solve_batch, group=None):
    """Batches of independent problems across GPUs (SURVEY.md 8(e) last item, 8(f) row 2): problem k
    goes to rank k % P -- replicas, no data-path collective -- each rank solves its share with
    `solve_batch(list_of_problems, cfg)` (Context.estimate_batch on the rank's GPU: worker streams)
    and one object all-gather gives every rank all results in problem order."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = list(range(rank, len(problems), world))
    results = solve_batch([problems[k] for k in mine], cfg) if mine else []
    gathered = [None] * world
    dist.all_gather_object(gathered, list(zip(mine, results)), group=group)
    out = [None] * len(problems)
    for part in gathered:
        for k, r in part:
            out[k] = r
    return out


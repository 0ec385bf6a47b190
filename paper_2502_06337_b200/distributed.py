"""Sharded estimate_single over ranks (one process per GPU; torch.distributed is the plumbing).

SURVEY.md section 8(e): rank r owns the contiguous correspondence range [N*r/P, N*(r+1)/P).

  vote     every rank preprocesses and votes its shard into a local uint32 grid; one all-reduce
           sums the grids (NCCL over NVLink on B200; integer sums, so the result is bit-identical
           to the single-GPU grid -- the reference's own chunked vote relies on the same property,
           voting.cpp:102-117)
  peak     every rank finds the same peak and start axis on the summed grid
           (estimate_from_peak, estimator.cpp:94-97)
  refine   refine_loop (estimator.cpp:51-69), sharded: each pass every rank classifies its own
           constraints and contributes 8 doubles (inlier count, "set changed", the 6 scatter sums
           of refine_axis), summed in rank order; every rank runs the same 3x3 solve -- identical
           axis and decision everywhere. With one GPU per rank this is ONE device-resident loop
           per rank (rv_shard_refine): the partials travel through peer memory (line buffers
           shared by CUDA IPC), no host round trip per pass; otherwise (ranks sharing a GPU, the
           CPU backend) the passes are host-stepped with an all-gather each
  estimate build_estimate (estimator.cpp:73-92): the rank-ordered concatenation of the shard
           inlier lists is the reference's ascending list; the angle histograms are summed and
           peak_angle's window sums around the summed peak are gathered and summed in rank order

Only ~100 bytes per pass cross the interconnect after the grid. The branches that need every
constraint on one device -- the identity shortcuts (estimator.cpp:326-340), the exactness-guard
re-vote and the rescue path (:352-368) -- fall back to the replicated finish: all-gather the input
and finish from the summed grid (rare: never on C1-C3).

The compute is behind a small backend interface, so the same protocol runs on B200s
(`DeviceBackend`, the C-ABI) and, in the CPU test-suite, on the oracle over gloo.
"""
from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous shard [lo, hi) of rank `rank`."""
    return n * rank // world, n * (rank + 1) // world


class DeviceBackend:
    """B200 backend: the shard steps through the C-ABI on the rank's GPU.

    The context runs on torch's current stream of the rank's device, so its work is ordered after
    the collectives torch enqueued there (all-reduce, all-gather) and before anything torch enqueues
    later; the C-ABI calls return after their own device work has completed."""

    def __init__(self, ctx, device=None):
        self.ctx = ctx
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self._sync_stream()

    def _sync_stream(self):
        self.ctx.set_stream(torch.cuda.current_stream(self.device).cuda_stream)

    def vote_shard(self, shard: torch.Tensor, cfg):
        self._sync_stream()
        g = torch.empty((cfg.grid, cfg.grid), dtype=torch.int32, device=shard.device)  # uint32 bits
        kept = self.ctx.vote_shard(shard.data_ptr(), shard.shape[0], g.data_ptr(), cfg)
        self.shard = shard
        return g, kept

    def peak_start_axis(self, grid: torch.Tensor, cfg):
        self._sync_stream()
        return self.ctx.peak_start_axis(grid.data_ptr(), cfg)

    def classify(self, axis, cfg, slot: int, compare: bool):
        return self.ctx.shard_classify(axis, cfg.epsilon, slot, compare)

    def inliers(self, slot: int, offset: int, count: int) -> np.ndarray:
        return self.ctx.shard_inliers(slot, offset, count)

    def angle_hist(self, axis, cfg):
        return self.ctx.shard_angle_hist(axis, cfg)

    def angle_sums(self, bins_total, cfg) -> np.ndarray:
        return self.ctx.shard_angle_sums(bins_total, cfg)

    def finish(self, corrs: torch.Tensor, grid: torch.Tensor, cfg):
        self._sync_stream()
        return self.ctx.estimate_single_prevoted(corrs.data_ptr(), corrs.shape[0], grid.data_ptr(), cfg)

    def rodrigues(self, axis, angle):
        import paper_2502_06337_b200 as rv
        return rv.rodrigues(axis, angle)

    def axis_from_scatter(self, s6):
        import paper_2502_06337_b200 as rv
        return rv.axis_from_scatter(s6)

    @property
    def tensor_device(self):
        return self.device

    # ---- device-resident refine across the ranks (rv_shard_refine over CUDA IPC line buffers) ----
    def peer_refine_ready(self, group=None) -> bool:
        """Collective (first call): export this rank's line buffer, gather every rank's IPC handle and
        GPU, map the peers' buffers. Disabled (host-stepped passes) when two ranks share a GPU --
        their cooperative kernels would wait on each other -- or with more than 8 ranks."""
        key = id(group)
        cache = getattr(self, "_xready", {})
        if key in cache:
            return cache[key] is not None
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        ptr, handle = self.ctx.shard_lines_export()
        uuid = str(torch.cuda.get_device_properties(self.device).uuid)
        info = [None] * world
        dist.all_gather_object(info, (uuid, handle), group=group)
        lines = None
        if world <= 8 and len({u for u, _ in info}) == world:
            lines = [ptr if r == rank else self.ctx.shard_lines_open(info[r][1]) for r in range(world)]
        cache[key] = lines
        self._xready = cache
        self._xepoch = getattr(self, "_xepoch", 0)
        return lines is not None

    def device_refine(self, axis0, cfg, group=None):
        """refine_loop of all shards as one cooperative loop per rank, the per-pass partials exchanged
        through peer memory; every rank returns the same (axis, total count, this shard's count)."""
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        self._xepoch += 1  # the same sequence of solves on every rank
        ax, count, local, _, refits = self.ctx.shard_refine(axis0, cfg, world, rank, self._xready[id(group)],
                                                           self._xepoch)
        return ax, count, local, refits


def all_gather_rows(shard: torch.Tensor, n_total: int, group=None) -> torch.Tensor:
    """Rank-ordered concatenation of every rank's shard (shapes are known from shard_bounds)."""
    world = dist.get_world_size(group)
    sizes = [shard_bounds(n_total, world, r)[1] - shard_bounds(n_total, world, r)[0] for r in range(world)]
    width = max(sizes)
    on = torch.device("cpu") if dist.get_backend(group) == "gloo" else shard.device
    padded = torch.zeros((width,) + tuple(shard.shape[1:]), dtype=shard.dtype, device=on)
    padded[: shard.shape[0]] = shard
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.cat([p[:s] for p, s in zip(parts, sizes)]).to(shard.device)


def _comm_device(backend, group):
    """Where the small collective tensors live: the rank's GPU for NCCL, host memory for gloo."""
    return torch.device("cpu") if dist.get_backend(group) == "gloo" else backend.tensor_device


def _all_reduce_(t: torch.Tensor, group) -> None:
    """In-place sum; a CUDA tensor under gloo goes through host memory."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)


def _gather_f64(vals, device, group) -> np.ndarray:
    """All-gather a small float64 vector from every rank -> (world, k) array in rank order."""
    world = dist.get_world_size(group)
    t = torch.as_tensor(np.asarray(vals, dtype=np.float64), device=device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return torch.stack(parts).cpu().numpy()


def _gather_i32_varlen(vals: np.ndarray, counts, device, group) -> np.ndarray:
    world = dist.get_world_size(group)
    width = max(1, int(max(counts)))
    t = torch.zeros(width, dtype=torch.int32, device=device)
    if vals.size:
        t[: vals.size] = torch.as_tensor(vals, device=device)
    parts = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(parts, t, group=group)
    return np.concatenate([p[: int(c)].cpu().numpy() for p, c in zip(parts, counts)]) if world else vals


def replicated_finish(shard: torch.Tensor, n_total: int, grid: torch.Tensor, cfg, backend, group=None):
    """All-gather the input and finish from the summed grid on every rank (the rare branches)."""
    corrs = all_gather_rows(shard, n_total, group)
    return backend.finish(corrs, grid, cfg)


def sharded_estimate_single(shard: torch.Tensor, n_total: int, cfg, backend, group=None, stats: dict | None = None):
    """estimate_single over all ranks' shards; every rank returns the same estimate (equal to the
    single-device estimate: identical grid, peak and inlier set; rotation within 1e-3 deg)."""
    from paper_2502_06337_b200 import RotationEstimate

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    dev = _comm_device(backend, group)
    lo, _ = shard_bounds(n_total, world, rank)
    grid, kept = backend.vote_shard(shard, cfg)
    # ONE all-reduce carries the grid and the kept count (an extra int32 word: int32 wrap-around ==
    # uint32 sum for the grid; the total kept count is < 2^31)
    cells = grid.numel()
    buf = torch.empty(cells + 1, dtype=torch.int32, device=grid.device)
    buf[:cells].copy_(grid.reshape(-1))
    buf[cells] = int(kept)
    _all_reduce_(buf, group)
    grid = buf[:cells].view(grid.shape)
    n_kept = int(buf[cells].item())
    mode = "sharded"
    if stats is not None:
        stats["mode"] = mode
    if n_kept == 0 or (n_total - n_kept) * 10 >= n_total * 9:  # identity shortcuts need the dropped list
        if stats is not None:
            stats["mode"] = "replicated:identity"
        return replicated_finish(shard, n_total, grid, cfg, backend, group)
    axis, votes, total = backend.peak_start_axis(grid, cfg)
    if total != n_kept * cfg.theta_samples:  # exactness guard: the replicated finish re-votes
        if stats is not None:
            stats["mode"] = "replicated:guard"
        return replicated_finish(shard, n_total, grid, cfg, backend, group)

    def classify(ax, slot, compare):
        c, sc, diff = backend.classify(ax, cfg, slot, compare)
        rows = _gather_f64([c, 1.0 if diff else 0.0, *sc], dev, group)
        s6 = np.zeros(6)
        for r in range(world):  # rank order
            s6 = s6 + rows[r, 2:]
        return rows[:, 0].astype(np.int64), bool(rows[:, 1].any()), s6

    slot = 0
    if hasattr(backend, "device_refine") and backend.peer_refine_ready(group):
        # device-resident refine_loop: one cooperative loop per rank, partials through peer memory
        axis, total_count, local, passes = backend.device_refine(axis, cfg, group)
        if cfg.refine and total_count < 3.0 * (cfg.epsilon * n_kept):  # rescue (estimator.cpp:352-368)
            if stats is not None:
                stats["mode"] = "replicated:rescue"
            return replicated_finish(shard, n_total, grid, cfg, backend, group)
        if stats is not None:
            stats["mode"] = "sharded:device"
            stats["passes"] = passes
        # the shard counts ride the angle-histogram all-reduce (no separate gather)
        return _sharded_build(shard, n_total, cfg, backend, group, axis, None, 0, lo, world, rank, dev, stats,
                              votes, local_count=int(local), total_count=int(total_count))
    counts, _, s6 = classify(axis, slot, False)
    passes = 0
    if cfg.refine:
        for _ in range(10):  # refine_loop (estimator.cpp:51-69)
            if counts.sum() < 2:
                break
            try:
                nxt = backend.axis_from_scatter(s6)
            except Exception as e:  # RankDeficient: keep the current axis
                if type(e).__name__ != "RankDeficient":
                    raise
                break
            counts, changed, s6 = classify(nxt, 1 - slot, True)
            slot = 1 - slot
            axis = np.asarray(nxt, dtype=np.float64)
            passes += 1
            if not changed:
                break
        if counts.sum() < 3.0 * (cfg.epsilon * n_kept):  # rescue (estimator.cpp:352-368)
            if stats is not None:
                stats["mode"] = "replicated:rescue"
            return replicated_finish(shard, n_total, grid, cfg, backend, group)
    if stats is not None:
        stats["passes"] = passes
    return _sharded_build(shard, n_total, cfg, backend, group, axis, counts, slot, lo, world, rank, dev, stats,
                          votes)


def _sharded_build(shard, n_total, cfg, backend, group, axis, counts, slot, lo, world, rank, dev, stats, votes,
                   local_count=None, total_count=None):
    """build_estimate (estimator.cpp:73-92) over the shards: the rank-ordered concatenation of the
    shard inlier lists is the reference's ascending list; the angle histograms are summed and
    peak_angle's window sums around the summed peak are summed in rank order. `counts` (every
    shard's inlier count) may be None: then each rank's own count travels in the histogram's
    all-reduce (one-hot slot per rank), which the inlier gather needs first."""
    from paper_2502_06337_b200 import RotationEstimate

    mine = int(counts[rank]) if counts is not None else int(local_count)
    local = backend.inliers(slot, lo, mine)  # compacts this shard's inliers (the angle vote's input)
    bins, contrib = backend.angle_hist(axis, cfg)
    # ONE all-reduce: the angle histogram, the contributing count, and the shard counts
    extra = np.zeros(1 + world, np.int64)
    extra[0] = contrib
    extra[1 + rank] = mine
    bins_t = torch.as_tensor(np.concatenate([bins.astype(np.int64), extra]), device=dev)
    dist.all_reduce(bins_t, group=group)
    summed = bins_t.cpu().numpy()
    nb = len(bins)
    if counts is None:
        counts = summed[nb + 1:].astype(np.int64)
        if total_count is not None:
            assert int(counts.sum()) == total_count
    inliers = _gather_i32_varlen(local, counts, dev, group)
    if int(summed[nb]) == 0:
        from paper_2502_06337_b200.errors import NoVotes
        raise NoVotes("no correspondence produced an angle vote")
    hist = summed[:nb].astype(np.uint32)
    peak = int(np.argmax(hist))  # first maximum (angles.cpp:70-90)
    w = 2.0 * math.pi / cfg.angle_bins
    angle = -math.pi + (peak + 0.5) * w
    if cfg.refine:
        rows = _gather_f64(backend.angle_sums(hist, cfg), dev, group)
        s = c = 0.0
        for r in range(world):  # rank order
            s += float(rows[r, 0])
            c += float(rows[r, 1])
        if not (s == 0.0 and c == 0.0):
            angle = math.atan2(s, c)
            if angle <= -math.pi:
                angle += 2.0 * math.pi
    axis = np.asarray(axis, dtype=np.float64)
    return RotationEstimate(axis=axis, angle=angle, rotation=backend.rodrigues(axis, angle),
                            inliers=inliers.astype(np.int32), axis_votes=int(votes))


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

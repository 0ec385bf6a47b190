"""CPU, world sizes 2 and 3 over gloo: the sharded protocol of paper_2502_06337_b200.distributed
(contiguous shards, all-reduced uint32 grids, sharded refine_loop with rank-ordered
partial sums, rank-ordered inlier concatenation, summed angle histograms and window sums) with the
oracle as the compute backend. Checks the reduced grid is bit-identical to the single-process vote,
the finish really ran sharded (no re-vote, no input all-gather), degenerate pairs in one shard keep
global index order, and every rank returns the oracle's single-process estimate."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_06337_b200 import distributed as rvd
from paper_2502_06337_b200 import synth


class OracleBackend:
    """CPU stand-in for DeviceBackend (tests only): the shard steps on the oracle port, the 3x3
    solve / geometry through the library's host functions (no GPU needed for those)."""

    tensor_device = torch.device("cpu")

    def __init__(self):
        import oracle as orc
        import paper_2502_06337_b200 as rv
        self.orc = orc
        self.rv = rv
        self.port = orc.Oracle("port")
        self.last_grid = None
        self.finished_replicated = False
        self.cls = [None, None]

    def vote_shard(self, shard, cfg):
        self.corrs = shard.numpy()
        self.z, self.kept, _ = self.port.preprocess(self.corrs) if shard.shape[0] else (np.zeros((0, 3)), [], [])
        g = self.port.accumulate(self.z, cfg.grid, cfg.extent, cfg.theta_samples) if len(self.z) else \
            np.zeros((cfg.grid, cfg.grid), np.uint32)
        return torch.from_numpy(g.view(np.int32).copy()), len(self.z)

    def peak_start_axis(self, grid, cfg):
        g = grid.numpy().view(np.uint32).reshape(cfg.grid, cfg.grid)
        self.last_grid = g.copy()
        ix, iy, A, B, votes = self.port.find_peaks(g, 1, cfg.suppression_radius, 1, cfg.extent)[0]
        cs = 2.0 * cfg.extent / cfg.grid
        wsum = asum = bsum = 0.0  # interpolate_peak (estimator.cpp:32-47): dy outer, dx inner
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                x, y = ix + dx, iy + dy
                if 0 <= x < cfg.grid and 0 <= y < cfg.grid:
                    wv = float(g[y, x])
                    wsum += wv
                    asum += wv * (-cfg.extent + (x + 0.5) * cs)
                    bsum += wv * (-cfg.extent + (y + 0.5) * cs)
        if wsum > 0:
            A, B = asum / wsum, bsum / wsum
        u = self.rv.unproject(A, B)
        axis = self.rv.canonicalize(u / np.linalg.norm(u))
        return axis, int(votes), int(g.sum(dtype=np.uint64))

    def classify(self, axis, cfg, slot, compare):
        inl = self.port.classify_inliers(np.asarray(axis), self.z, cfg.epsilon) if len(self.z) else np.zeros(0, int)
        prev = self.cls[1 - slot]
        differs = compare and (prev is None or not np.array_equal(prev, inl))
        self.cls[slot] = inl
        zi = self.z[inl] if len(inl) else np.zeros((0, 3))
        sc = [float(np.sum(zi[:, a] * zi[:, b])) for a, b in ((0, 0), (0, 1), (0, 2), (1, 1), (1, 2), (2, 2))]
        return len(inl), np.array(sc), bool(differs)

    def inliers(self, slot, offset, count):
        self.idx = np.asarray(self.kept, dtype=np.int64)[self.cls[slot]] if count else np.zeros(0, np.int64)
        return (self.idx + offset).astype(np.int32)

    def angle_hist(self, axis, cfg):
        bins = np.zeros(cfg.angle_bins, np.uint32)
        self.raw = []
        w = 2.0 * math.pi / cfg.angle_bins
        for i in self.idx:  # vote_angles (angles.cpp:46-68)
            c = self.corrs[i]
            try:
                a = self.rv.correspondence_angle(axis, c[:3], c[3:], cfg.tau_deg)
            except Exception:
                continue
            k = min(max(int(math.ceil((a + math.pi) / w)) - 1, 0), cfg.angle_bins - 1)
            bins[k] += 1
            self.raw.append(a)
        return bins, len(self.raw)

    def angle_sums(self, bins_total, cfg):
        w = 2.0 * math.pi / cfg.angle_bins
        center = -math.pi + (int(np.argmax(bins_total)) + 0.5) * w
        s = c = 0.0
        for a in self.raw:  # peak_angle's window (angles.cpp:70-90)
            d = math.fmod(a - center, 2.0 * math.pi)
            if d <= -math.pi:
                d += 2.0 * math.pi
            if d > math.pi:
                d -= 2.0 * math.pi
            if abs(d) <= 1.5 * w:
                s += math.sin(a)
                c += math.cos(a)
        return np.array([s, c])

    def axis_from_scatter(self, s6):
        return self.rv.axis_from_scatter(s6)

    def rodrigues(self, axis, angle):
        return self.rv.rodrigues(axis, angle)

    def finish(self, corrs, grid, cfg):
        self.finished_replicated = True
        self.last_grid = grid.numpy().view(np.uint32).copy()
        r = self.port.estimate_single(corrs.numpy(), self.orc.default_config())
        return self.rv.RotationEstimate(axis=r["axis"], angle=r["angle"], rotation=r["rotation"],
                                        inliers=r["inliers"], axis_votes=r["axis_votes"])


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def worker(rank, world, port, corrs, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root / "oracle"))
    import paper_2502_06337_b200 as rv
    lo, hi = rvd.shard_bounds(corrs.shape[0], world, rank)
    backend = OracleBackend()
    shard = torch.from_numpy(corrs[lo:hi].copy())
    stats = {}
    est = rvd.sharded_estimate_single(shard, corrs.shape[0], rv.EstimatorConfig(), backend, stats=stats)
    out[rank] = (backend.last_grid.reshape(-1), est.inliers, est.rotation, est.axis_votes, stats.get("mode"),
                 backend.finished_replicated)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_protocol_matches_single_process(world):
    import oracle as orc
    corrs, _, _ = synth.make_scene(3001, 0.7, 0.01, seed=4242)
    corrs[5, 3:] = corrs[5, :3]          # degenerate pairs (dropped) in the first shard ...
    corrs[2999, 3:] = corrs[2999, :3]    # ... and the last
    port = orc.Oracle("port")
    z, kept, dropped = port.preprocess(corrs)
    assert dropped.tolist() == [5, 2999]
    ref_grid = port.accumulate(z)
    ref = port.estimate_single(corrs)
    out = mp.Manager().dict()
    mp.spawn(worker, args=(world, free_port(), corrs, out), nprocs=world, join=True)
    for r in range(world):
        grid, inl, rot, votes, mode, replicated = out[r]
        assert mode == "sharded" and not replicated, f"rank {r}: finish did not run sharded ({mode})"
        assert np.array_equal(grid, ref_grid.reshape(-1)), f"rank {r}: reduced grid differs"
        assert np.array_equal(inl, ref["inliers"]), f"rank {r}: inlier set differs"
        assert orc.rotation_error_deg(rot, ref["rotation"]) <= 1e-3
        assert votes == ref["axis_votes"]


def test_shard_bounds_partition():
    for n in (0, 1, 7, 1000, 1_000_001):
        for world in (1, 2, 3, 8):
            b = [rvd.shard_bounds(n, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))


def batch_worker(rank, world, port, problems, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path.insert(0, str(root / "oracle"))
    import oracle as orc
    port_ = orc.Oracle("port")
    solve = lambda ps, cfg: [port_.estimate_single(p) for p in ps]  # noqa: E731 (CPU stand-in)
    res = rvd.batch_estimate(problems, None, solve)
    out[rank] = [(r["inliers"], r["rotation"]) for r in res]
    dist.destroy_process_group()


def test_batch_round_robin_across_ranks():
    import sys
    from pathlib import Path
    sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "oracle"))
    import oracle as orc
    problems = [synth.make_scene(400, 0.5, 0.01, seed=700 + k)[0] for k in range(5)]
    ref = [orc.Oracle("port").estimate_single(p) for p in problems]
    world = 2
    out = mp.Manager().dict()
    mp.spawn(batch_worker, args=(world, free_port(), problems, out), nprocs=world, join=True)
    for rank in range(world):
        assert len(out[rank]) == len(problems)
        for (inl, rot), r in zip(out[rank], ref):
            assert np.array_equal(inl, r["inliers"]) and np.array_equal(rot, r["rotation"])


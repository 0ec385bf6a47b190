"""CPU, world_size 2 over gloo: the sharded protocol of paper_2502_06337_b200.distributed
(contiguous shards, all-reduced uint32 grids, rank-ordered all-gather, replicated finish) with
the oracle as the compute backend. Checks the reduced grid is bit-identical to the single-process
vote, degenerate pairs in one shard keep global index order, and both ranks return the oracle's
single-process estimate."""
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
    """CPU stand-in for DeviceBackend (tests only): the oracle votes and finishes."""

    def __init__(self):
        import oracle as orc
        self.orc = orc
        self.port = orc.Oracle("port")
        self.last_grid = None

    def vote_shard(self, shard, cfg):
        z, kept, dropped = self.port.preprocess(shard.numpy())
        g = self.port.accumulate(z, cfg.grid, cfg.extent, cfg.theta_samples) if len(z) else \
            np.zeros((cfg.grid, cfg.grid), np.uint32)
        return torch.from_numpy(g.view(np.int32).copy())

    def finish(self, corrs, grid, cfg):
        self.last_grid = grid.numpy().view(np.uint32).copy()
        return self.port.estimate_single(corrs.numpy(), self.orc.default_config())


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
    est = rvd.sharded_estimate_single(shard, corrs.shape[0], rv.EstimatorConfig(), backend)
    out[rank] = (backend.last_grid, est["inliers"], est["rotation"], est["axis_votes"])
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
        grid, inl, rot, votes = out[r]
        assert np.array_equal(grid, ref_grid), f"rank {r}: reduced grid differs"
        assert np.array_equal(inl, ref["inliers"]) and np.array_equal(rot, ref["rotation"])
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


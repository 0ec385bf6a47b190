"""GPU tests of the multi-GPU paths on the one B200 a test box has.

* rv_multi (one process, NCCL clique via ncclCommInitAll) over a one-device list: the same
  sharded code -- shard vote, in-place ncclAllReduce of the u32 grid, sharded refine / angle
  finish -- must reproduce the reference's full-size goldens (C3 at N = 1e6) and the
  single-device grid, and the rescue branch (C4) must hand over to device 0 correctly.
* distributed.sharded_estimate_single (one process per GPU) with a world-1 NCCL group, and with
  two ranks on one GPU over gloo (host collectives: no kernel of one rank waits on the other's).
* the reference's own unit suites through the C++ drop-in with ROTAVOTE_DEVICES set (the rv_multi
  route of rotavote::estimate_single / accumulate).
"""
import os
import socket
import subprocess
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle as orc
import paper_2502_06337_b200 as rv
from conftest import golden
from paper_2502_06337_b200 import distributed as rvd
from paper_2502_06337_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def check_golden(e, g, prefix="est_"):
    assert np.array_equal(e.inliers, g[f"{prefix}inliers"]), "inlier sets differ"
    assert e.axis_votes == int(g[f"{prefix}axis_votes"])
    assert orc.rotation_error_deg(e.rotation, g[f"{prefix}rotation"]) <= 1e-3


@pytest.fixture(scope="module")
def multi():
    return rv.MultiContext([0])


def test_multi_context_nccl_clique(multi):
    assert multi.nccl_version >= 21800  # ncclCommInitAll ran (NCCL 2.18+)


def test_multi_estimate_single_c3_fullsize(multi):
    g = golden("c3_full")
    corrs, _, _ = synth.make_config("c3")
    e = multi.estimate_single(corrs)
    check_golden(e, g)


def test_multi_estimate_single_rescue_and_identity(multi, ctx):
    # C4 takes the rescue branch: the multi path hands the summed grid to device 0
    g = golden("c4_full")
    corrs, _, _ = synth.make_config("c4")
    check_golden(multi.estimate_single(corrs), g)
    # >= 90% degenerate pairs: identity with the dropped list, like the single-device path
    small, _, _ = synth.make_scene(5000, 0.5, 0.01, seed=137)
    small[:4600, 3:] = small[:4600, :3]
    e = multi.estimate_single(small)
    assert np.allclose(e.rotation, np.eye(3)) and np.array_equal(e.inliers, np.arange(4600))


def test_multi_accumulate_matches_single(multi, ctx):
    rng = np.random.default_rng(11)
    z = rng.normal(size=(20000, 3))
    z /= np.linalg.norm(z, axis=1, keepdims=True)
    assert np.array_equal(multi.accumulate(z), ctx.accumulate(z))


def test_sharded_protocol_world1_nccl(ctx):
    # one-rank NCCL group: every step of the sharded finish runs on the device
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(free_port()))
    dist.init_process_group("nccl", rank=0, world_size=1)
    try:
        g = golden("c3_full")
        corrs, _, _ = synth.make_config("c3")
        d = torch.from_numpy(corrs).cuda()
        stats = {}
        e = rvd.sharded_estimate_single(d, corrs.shape[0], rv.EstimatorConfig(), rvd.DeviceBackend(ctx), stats=stats)
        # one GPU per rank: the refine runs device-resident (rv_shard_refine over the ranks' line
        # buffers exported / mapped by CUDA IPC; one rank here, so its own buffer only)
        assert stats["mode"] == "sharded:device" and stats["passes"] >= 1
        check_golden(e, g)
    finally:
        dist.destroy_process_group()


def gloo_worker(rank, world, port, n, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    corrs, _, _ = synth.make_config("c3", n)
    lo, hi = rvd.shard_bounds(n, world, rank)
    ctx = rv.Context(0)
    shard = torch.from_numpy(np.ascontiguousarray(corrs[lo:hi])).cuda()
    stats = {}
    e = rvd.sharded_estimate_single(shard, n, rv.EstimatorConfig(), rvd.DeviceBackend(ctx, 0), stats=stats)
    out[rank] = (e.inliers, e.rotation, e.axis_votes, stats["mode"], stats.get("passes", 0))
    dist.destroy_process_group()


def test_sharded_protocol_two_ranks_one_gpu(ctx):
    n = 200_000
    corrs, _, _ = synth.make_config("c3", n)
    ref = ctx.estimate_single(corrs)
    out = mp.get_context("spawn").Manager().dict()
    mp.spawn(gloo_worker, args=(2, free_port(), n, out), nprocs=2, join=True)
    for r in range(2):
        inl, rot, votes, mode, passes = out[r]
        # two ranks on ONE GPU: their cooperative kernels must not wait on each other, so the
        # passes are host-stepped (peer_refine_ready sees the same GPU twice)
        assert mode == "sharded" and passes >= 1
        assert np.array_equal(inl, ref.inliers) and votes == ref.axis_votes
        assert orc.rotation_error_deg(rot, ref.rotation) <= 1e-3


def test_dropin_reference_suites_through_multi():
    import re
    exe = ROOT / "tests" / "_bin" / "ref_tests_on_b200"
    if not exe.exists():
        pytest.skip("drop-in binary not built (tests/dropin: make)")
    env = dict(os.environ, ROTAVOTE_DEVICES="0")  # estimate_single / accumulate via rv_multi
    r = subprocess.run([str(exe)], capture_output=True, text=True, env=env, timeout=600)
    out = r.stdout + r.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| assertions: (\d+) \| (\d+) failed", out)
    assert m, out[-2000:]
    cases, passed, failed, asserts, afailed = map(int, m.groups())
    assert failed == 0 and afailed == 0 and cases >= 50, out[-3000:]


def test_shard_refine_device_resident_matches_single(ctx):
    # rv_shard_refine (the cooperative refine_loop of a shard, whose per-pass partials go through
    # peer memory on a multi-GPU box) with one device: the same loop, the same fixed-order sums and
    # the same final set as the single-device solve, bit for bit
    corrs, _, _ = synth.make_config("c3", 200_000)
    cfg = rv.EstimatorConfig()
    d = torch.from_numpy(corrs).cuda()
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    try:
        grid = torch.zeros((cfg.grid, cfg.grid), dtype=torch.int32, device="cuda")
        kept = ctx.vote_shard(d.data_ptr(), corrs.shape[0], grid.data_ptr(), cfg)
        axis0, _, total = ctx.peak_start_axis(grid.data_ptr(), cfg)
        assert total == kept * cfg.theta_samples
        ax, count, local, scatter, refits = ctx.shard_refine(axis0, cfg)
        assert count == local and refits >= 1
        inl = ctx.shard_inliers(0, 0, count)
        e = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
        assert np.array_equal(inl, e.inliers)
        assert np.array_equal(ax, e.axis)
    finally:
        ctx.set_stream(None)

"""GPU parity: the sm_100a path, called through the C-ABI, against the CPU oracle and the
reference's golden vectors. Bar (BASELINE.json north star): vote grids bit-exact, peaks and
inlier sets identical, rotations within 1e-3 degrees (they are in fact identical or ~1e-6 deg:
only the parallel order of the 6 scatter sums differs from the reference's sequential sum).
"""
import hashlib

import numpy as np
import pytest

import oracle as orc
import paper_2502_06337_b200 as rv
from conftest import golden
from paper_2502_06337_b200 import synth

pytestmark = pytest.mark.gpu
ROT_TOL_DEG = 1e-3


def unit_rows(rng, n):
    z = rng.normal(size=(n, 3))
    return z / np.linalg.norm(z, axis=1, keepdims=True)


def assert_est_equal(dev, ref: dict):
    assert np.array_equal(dev.inliers, ref["inliers"]), "inlier sets differ"
    assert dev.axis_votes == ref["axis_votes"]
    assert orc.rotation_error_deg(dev.rotation, ref["rotation"]) <= ROT_TOL_DEG
    assert np.allclose(dev.axis, ref["axis"], atol=1e-12)


# ---- vote grid (voting.cpp:88-118): bit-exact for every configuration -----------------------
@pytest.mark.parametrize("grid,extent,samples", [
    (512, 1.05, 2048),   # reference default (band-tiled smem kernel)
    (256, 1.05, 1024),   # reference unit-test "small_cfg"
    (128, 1.05, 512),    # deposit tests
    (512, 1.05, 1000),   # J not a multiple of 128 -> exact generic kernel
    (97, 1.3, 640),      # odd grid, wide extent
    (200, 0.9, 1024),    # extent < 1: clamped cells
    (1024, 1.05, 4096),  # finer grid, more bands (run-time fixed-point shift S=11)
    (1100, 0.95, 1024),  # clamped cells with the run-time shift
    (256, 0.5, 1024),    # small extent: clamped, compile-time S=13
    (512, 0.2, 1024),    # very small extent: large cell scale K -> run-time S=10
])
def test_accumulate_bit_exact(ctx, port, grid, extent, samples):
    rng = np.random.default_rng(grid + samples)
    z = unit_rows(rng, 3000)
    assert np.array_equal(ctx.accumulate(z, grid, extent, samples), port.accumulate(z, grid, extent, samples))


def test_accumulate_bit_exact_large_default(ctx, port):
    # the f32 filter's error budget is tightest at the default geometry (S=13): 40k random
    # constraints = 41M sampled pairs against the oracle
    rng = np.random.default_rng(20250206)
    z = unit_rows(rng, 40000)
    assert np.array_equal(ctx.accumulate(z), port.accumulate(z))


def test_accumulate_adversarial_constraints(ctx, port):
    # axis-aligned, polar, horizontal/vertical diameters, near-polar, duplicated constraints
    special = [[0, 0, 1], [0, 0, -1], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0],
               [1, 1, 0], [1, 0, 1], [0, 1, 1], [1e-7, 0, 1], [1e-4, 1e-4, 1], [0.6, 0.8, 0],
               [1, 1, 1], [-1, 1, 1e-12], [3e-4, 0, 1]]
    z = np.array(special, dtype=np.float64)
    z /= np.linalg.norm(z, axis=1, keepdims=True)
    z = np.concatenate([z, z[:5]])
    for grid, samples in ((512, 2048), (256, 1024), (128, 512)):
        assert np.array_equal(ctx.accumulate(z, grid, 1.05, samples), port.accumulate(z, grid, 1.05, samples))


def tangent_constraints(grid: int, extent: float) -> np.ndarray:
    """Great circles whose projected arc is tangent (from above and below) to EVERY grid row
    boundary Y = -E + r * 2E/G inside the unit disk: the planner's band boundaries are among them,
    and a tangent visit is its ill-conditioned case. The image of the great circle with unit normal
    n is the circle of centre -(nx, ny)/nz and radius 1/|nz| (stereographic projection)."""
    out = []
    cs = 2.0 * extent / grid
    for r in range(1, grid):
        y0 = -extent + r * cs
        if abs(y0) >= 0.999 or abs(y0) < 1e-9:
            continue
        for cx in (0.0, 0.4 * np.sqrt(1.0 - y0 * y0)):
            for top in (True, False):  # the circle's top (bottom) point touches Y = y0
                cy = (y0 * y0 - 1.0 - cx * cx) / (2.0 * y0) if top else (1.0 + cx * cx - y0 * y0) / (2.0 * y0)
                rad = np.sqrt(1.0 + cx * cx + cy * cy)
                if (top and not (y0 - cy > 0)) or (not top and not (cy - y0 > 0)) or abs(abs(cy + (rad if top else -rad)) - abs(y0)) > 1e-9:
                    continue
                nz = 1.0 / rad
                out.append([-cx * nz, -cy * nz, nz])
    z = np.array(out)
    return z / np.linalg.norm(z, axis=1, keepdims=True)


@pytest.mark.parametrize("grid,extent,samples", [(512, 1.05, 2048), (256, 1.05, 1024), (1024, 1.05, 4096),
                                                 (200, 0.9, 1024)])
def test_accumulate_row_boundary_tangents(ctx, port, grid, extent, samples):
    # tangent visits of every row boundary (so of every band boundary) plus z = +-e2, whose arc is
    # the row boundary Y = 0 itself when G/2 is a band boundary; with RV_STRICT_GUARD a coverage
    # gap of the band plan is an error, not a silent exact re-vote
    z = np.concatenate([tangent_constraints(grid, extent), [[0.0, 1.0, 0.0], [0.0, -1.0, 0.0]]])
    assert z.shape[0] > grid
    assert np.array_equal(ctx.accumulate(z, grid, extent, samples), port.accumulate(z, grid, extent, samples))


@pytest.mark.parametrize("key", ["c1", "c2", "c3", "c4", "c5"])
def test_config_golden(ctx, key):
    g = golden(key)
    corrs, _, _ = synth.make_config(key, int(g["n"]))
    z, kept, _ = ctx.preprocess(corrs)
    assert hashlib.sha256(z.tobytes()).digest() == bytes(g["z_sha256"])
    grid = ctx.accumulate(z)
    assert hashlib.sha256(grid.tobytes()).digest() == bytes(g["grid_sha256"])
    peaks = ctx.find_peaks(grid, 3, 8, 1)
    assert [[p.ix, p.iy, p.votes] for p in peaks] == g["peaks"].tolist()
    for (w, b) in zip((4, 8, 16, 32, 64), g["blur"].tolist()):
        p = ctx.blurred_argmax(grid, w)
        assert [p.ix, p.iy, p.votes] == b
    if key == "c5":
        ms = ctx.estimate_multi(corrs, rv.EstimatorConfig(max_models=3))
        assert len(ms) == int(g["n_models"])
        for k, m in enumerate(ms):
            assert_est_equal(m, {"inliers": g[f"m{k}_inliers"], "axis_votes": int(g[f"m{k}_axis_votes"]),
                                 "rotation": g[f"m{k}_rotation"], "axis": g[f"m{k}_axis"]})
    else:
        e = ctx.estimate_single(corrs)
        assert_est_equal(e, {"inliers": g["est_inliers"], "axis_votes": int(g["est_axis_votes"]),
                             "rotation": g["est_rotation"], "axis": g["est_axis"]})


def test_fixture300(ctx):
    g = golden("fixture300")
    e = ctx.estimate_single(g["corrs"])
    assert_est_equal(e, {"inliers": g["est_inliers"], "axis_votes": int(g["est_axis_votes"]),
                         "rotation": g["est_rotation"], "axis": g["est_axis"]})
    assert abs(orc.rotation_error_deg(g["r_truth"], e.rotation) - 0.271442) < 1e-3


# ---- solver parity at larger sizes (oracle finishes in seconds) -----------------------------
@pytest.mark.parametrize("key,n", [("c1", 1000), ("c2", 100_000), ("c3", 200_000), ("c4", 200_000)])
def test_estimate_single_parity(ctx, port, key, n):
    corrs, rots, _ = synth.make_config(key, n)
    e = ctx.estimate_single(corrs)
    r = port.estimate_single(corrs)
    assert_est_equal(e, r)


def test_estimate_multi_parity(ctx, port):
    corrs, rots, _ = synth.make_config("c5", 200_000)
    ms = ctx.estimate_multi(corrs, rv.EstimatorConfig(max_models=3))
    rs = port.estimate_multi(corrs, orc.default_config(max_models=3))
    assert len(ms) == len(rs) == 3
    for m, r in zip(ms, rs):
        assert_est_equal(m, r)


def test_small_cfg_and_unrefined(ctx, port):
    corrs, _, _ = synth.make_scene(4000, 0.5, 0.01, seed=77)
    for cfg_kw in ({"grid": 256, "theta_samples": 1024}, {"refine": False}, {"normalize_inputs": False},
                   {"epsilon": 0.03, "angle_bins": 64}):
        e = ctx.estimate_single(corrs, rv.EstimatorConfig(**cfg_kw))
        r = port.estimate_single(corrs, orc.default_config(**cfg_kw))
        assert_est_equal(e, r)


# ---- path functions ------------------------------------------------------------------------
def test_preprocess_drops_and_errors(ctx, port):
    rng = np.random.default_rng(67)
    x = unit_rows(rng, 10)
    y = unit_rows(rng, 10)
    y[::3] = x[::3]
    corrs = np.concatenate([x, y], axis=1)
    zd, kd, dd = ctx.preprocess(corrs, 1e-9, False)
    zr, kr, dr = port.preprocess(corrs, 1e-9, False)
    assert np.array_equal(zd.view(np.uint64), zr.view(np.uint64))
    assert np.array_equal(kd, kr) and np.array_equal(dd, dr) and dd.tolist() == [0, 3, 6, 9]
    with pytest.raises(rv.AllDegenerate):
        ctx.preprocess(np.concatenate([x, x], axis=1), 1e-9, False)


def test_find_peaks_nms_and_mirror(ctx, port):
    rng = np.random.default_rng(13)
    axis_a = np.array([0.1, 0.2, -0.97])
    axis_a /= np.linalg.norm(axis_a)
    axis_b = rv.rodrigues([1, 0, 0], np.pi / 4) @ axis_a
    axis_c = np.array([0.8, 0.6, 0.0])  # equatorial axis: mirror suppression path
    z = []
    for ax, cnt in ((axis_a, 50), (axis_b, 60), (axis_c, 70)):
        a1, a2 = rv.orthonormal_basis(ax)
        t = rng.uniform(-np.pi, np.pi, cnt)
        z.append(np.outer(np.cos(t), a1) + np.outer(np.sin(t), a2))
    z = np.concatenate(z + [unit_rows(rng, 100)])
    grid = port.accumulate(z)
    for k, r, mv in ((1, 8, 1), (2, 8, 40), (3, 8, 1), (6, 4, 1), (8, 16, 10)):
        dev = ctx.find_peaks(grid, k, r, mv)
        ref = port.find_peaks(grid, k, r, mv)
        assert [(p.ix, p.iy, p.votes) for p in dev] == [(p[0], p[1], p[4]) for p in ref]
    with pytest.raises(rv.NoPeak):
        ctx.find_peaks(np.zeros((64, 64), np.uint32), 1, 4, 1)


def test_find_peaks_any_k(ctx, port):
    # the reference's find_peaks takes any max_peaks (voting.cpp:120-170): beyond the argmax
    # kernel's direct disks the suppression becomes a device bit image; K = 40 on a busy grid,
    # several radii, mirrors included, must match the oracle peak for peak
    corrs, _, _ = synth.make_config("c5", 20_000)
    z, _, _ = port.preprocess(corrs)
    grid = port.accumulate(z)
    for k, r, mv in ((40, 8, 1), (25, 3, 1), (60, 16, 1), (30, 6, 500)):
        dev = ctx.find_peaks(grid, k, r, mv)
        ref = port.find_peaks(grid, k, r, mv)
        assert [(p.ix, p.iy, p.votes) for p in dev] == [(p[0], p[1], p[4]) for p in ref]
    # an equatorial ring of peaks: every peak brings its mirror disk
    g = np.zeros((128, 128), np.uint32)
    for t in range(24):
        a = 2 * np.pi * t / 24
        g[int(64 + 60 * np.sin(a)), int(64 + 60 * np.cos(a))] = 100 + t
    dev = ctx.find_peaks(g, 24, 2, 1)
    ref = port.find_peaks(g, 24, 2, 1)
    assert [(p.ix, p.iy, p.votes) for p in dev] == [(p[0], p[1], p[4]) for p in ref]


def test_blurred_argmax_ties_and_edges(ctx, port):
    g = np.zeros((64, 64), np.uint32)
    g[0, 0] = 5
    g[63, 63] = 5
    g[10, 50] = 3
    for r in (0, 1, 4, 31, 64):
        p = ctx.blurred_argmax(g, r)
        q = port.blurred_argmax(g, r)
        assert (p.ix, p.iy, p.votes) == (q[0], q[1], q[4])
    with pytest.raises(rv.InvalidConfig):
        ctx.blurred_argmax(g, -1)


def test_classify_refine_angles(ctx, port):
    rng = np.random.default_rng(71)
    z = unit_rows(rng, 50_000)
    axis = rv.canonicalize(unit_rows(rng, 1)[0])
    assert np.array_equal(ctx.classify_inliers(axis, z, 0.015), port.classify_inliers(axis, z, 0.015))
    zb = np.array([[np.sqrt(1 - 0.015 ** 2), 0, 0.015]])
    assert ctx.classify_inliers([0, 0, 1.0], zb, 0.015).size == 0
    a = ctx.refine_axis(z[:1000])
    b = port.refine_axis(z[:1000])
    assert np.allclose(a, b, atol=1e-12)
    with pytest.raises(rv.RankDeficient):
        ctx.refine_axis(np.array([[1.0, 0, 0], [-1.0, 0, 0]]))
    # vote_angles / peak_angle (angles.cpp): noiseless votes land in one bin; refine is exact
    ax = rv.canonicalize(unit_rows(rng, 1)[0])
    R = rv.rodrigues(ax, np.deg2rad(30))
    x = unit_rows(rng, 60)
    corrs = np.concatenate([x, x @ R.T], axis=1)
    h = ctx.vote_angles(ax, corrs, np.arange(60), 64)
    assert h["contributing"] + h["degenerate"] == 60 and h["bins"].max() == h["contributing"]
    assert abs(ctx.peak_angle(h, True) - np.deg2rad(30)) < 1e-12
    with pytest.raises(rv.NoVotes):
        ctx.vote_angles(ax, corrs, np.zeros(0, np.int32), 64)


def test_deposit_circle_votes(ctx, port):
    g = np.zeros((128, 128), np.uint32)
    ctx.deposit_circle_votes([0, 0, 1.0], g, 1.05, 512)
    assert g.sum() == 512
    assert np.array_equal(g, port.accumulate(np.array([[0, 0, 1.0]]), 128, 1.05, 512))


def test_estimate_errors_and_identity(ctx):
    with pytest.raises(rv.EmptyInput):
        ctx.estimate_single(np.zeros((0, 6)))
    rng = np.random.default_rng(79)
    x = unit_rows(rng, 20)
    e = ctx.estimate_single(np.concatenate([x, x], axis=1))
    assert np.allclose(e.rotation, np.eye(3)) and e.inliers.size == 20
    with pytest.raises(rv.NoPeak):
        corrs, _, _ = synth.make_scene(2000, 1.0, 0.0, seed=109)
        ctx.estimate_multi(corrs, rv.EstimatorConfig(max_models=2))


# ---- full BASELINE sizes: size-independent properties ---------------------------------------
@pytest.mark.parametrize("key", ["c3", "c4"])
def test_full_size_properties(ctx, key):
    corrs, rots, labels = synth.make_config(key)
    e1 = ctx.estimate_single(corrs)
    e2 = ctx.estimate_single(corrs)
    assert np.array_equal(e1.inliers, e2.inliers) and np.array_equal(e1.rotation, e2.rotation)  # deterministic
    z, kept, _ = ctx.preprocess(corrs)
    grid = ctx.accumulate(z)
    assert int(grid.sum(dtype=np.uint64)) == z.shape[0] * 2048  # every sample counted exactly once
    a = e1.axis
    d = np.abs(z[:, 0] * a[0] + z[:, 1] * a[1] + z[:, 2] * a[2])  # reference op order, no FMA
    assert np.array_equal(np.nonzero(d < 0.015)[0], e1.inliers)  # inliers == strict predicate
    assert orc.rotation_error_deg(rots[0], e1.rotation) < (0.05 if key == "c3" else 1.0)


def test_beyond_c3_size_properties(ctx):
    # N = 3e6: the cooperative refine's per-block slice no longer fits shared memory (global-load
    # path), the pipelined host path runs 4 large chunks; size-independent properties hold
    import torch
    corrs, rots, _ = synth.make_config("c3", 3_000_000)
    d = torch.from_numpy(corrs).cuda()
    e_dev = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0])
    e_host = ctx.estimate_single(corrs)
    assert np.array_equal(e_dev.inliers, e_host.inliers) and np.array_equal(e_dev.rotation, e_host.rotation)
    z, kept, _ = ctx.preprocess(corrs)
    a = e_dev.axis
    dd = np.abs(z[:, 0] * a[0] + z[:, 1] * a[1] + z[:, 2] * a[2])
    assert np.array_equal(kept[np.nonzero(dd < 0.015)[0]], e_dev.inliers)  # strict predicate, input order
    grid = ctx.accumulate(z)
    assert int(grid.sum(dtype=np.uint64)) == z.shape[0] * 2048
    assert orc.rotation_error_deg(rots[0], e_dev.rotation) < 0.05
    assert ctx.stage_times()["vote_guard_reruns"] == 0


def test_pipelined_host_path_matches_device_path(ctx):
    # estimate_single with host input overlaps chunked H2D with preprocess/plan/vote; the result
    # must be identical to the device-resident solve (same grid => same peak, inliers, rotation)
    import torch
    corrs, _, _ = synth.make_config("c3")
    e_host = ctx.estimate_single(corrs)
    d = torch.from_numpy(corrs).cuda()
    e_dev = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0])
    assert np.array_equal(e_host.inliers, e_dev.inliers) and np.array_equal(e_host.rotation, e_dev.rotation)
    assert e_host.axis_votes == e_dev.axis_votes
    st = ctx.stage_times()
    assert st["vote_guard_reruns"] == 0


def test_inorder_path_with_dropped_pairs(ctx, port):
    # single solves keep the constraint set in input order (z = NaN marks a dropped pair); with
    # 20% scattered degenerate pairs the pipelined host path (4 chunks), the device path and the
    # oracle must agree, and >= 90% dropped takes the identity shortcut with the dropped list
    import torch
    corrs, _, _ = synth.make_config("c3", 300_000)
    rng = np.random.default_rng(131)
    drop = rng.random(corrs.shape[0]) < 0.2
    corrs[drop, 3:] = corrs[drop, :3]
    e_host = ctx.estimate_single(corrs)
    d = torch.from_numpy(corrs).cuda()
    e_dev = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0])
    r = port.estimate_single(corrs)
    assert_est_equal(e_host, r)
    assert_est_equal(e_dev, r)
    assert not np.isin(e_host.inliers, np.nonzero(drop)[0]).any()
    small, _, _ = synth.make_scene(5000, 0.5, 0.01, seed=137)
    small[:4600, 3:] = small[:4600, :3]
    e = ctx.estimate_single(small)
    assert np.allclose(e.rotation, np.eye(3)) and np.array_equal(e.inliers, np.arange(4600))
    assert np.array_equal(e.inliers, port.estimate_single(small)["inliers"])


def test_graph_replay_of_device_solves(ctx, port):
    # repeated device-resident solves with the same (pointer, n, config) replay a captured CUDA
    # graph; results must equal the eager solve, follow new data written to the same buffer, and
    # survive buffer reallocations in between (the graph is re-captured, never replayed stale)
    import torch
    a, _, _ = synth.make_config("c3", 300_000)
    b, _, _ = synth.make_scene(300_000, 0.5, 0.01, seed=149)
    d = torch.from_numpy(a).cuda()
    runs = [ctx.estimate_single_device(d.data_ptr(), a.shape[0]) for _ in range(4)]
    for e in runs[1:]:
        assert np.array_equal(e.inliers, runs[0].inliers) and np.array_equal(e.rotation, runs[0].rotation)
    assert_est_equal(runs[-1], port.estimate_single(a))
    d.copy_(torch.from_numpy(b))  # new contents, same pointer: the replay must see them
    eb = ctx.estimate_single_device(d.data_ptr(), b.shape[0])
    assert_est_equal(eb, port.estimate_single(b))
    # pinned host input: the pipelined solve (chunked H2D + chain) is captured and replayed too
    h = torch.empty((a.shape[0], 6), dtype=torch.float64, pin_memory=True)
    h.numpy()[:] = a
    hr = [ctx.estimate_single(h.numpy()) for _ in range(4)]
    for e in hr:
        assert np.array_equal(e.inliers, runs[0].inliers) and np.array_equal(e.rotation, runs[0].rotation)
    h.numpy()[:] = b
    eh = ctx.estimate_single(h.numpy())
    assert np.array_equal(eh.inliers, eb.inliers) and np.array_equal(eh.rotation, eb.rotation)
    big, _, _ = synth.make_config("c3")  # larger solve: grows (reallocates) the context buffers
    db = torch.from_numpy(big).cuda()
    ctx.estimate_single_device(db.data_ptr(), big.shape[0])
    for _ in range(3):
        e = ctx.estimate_single_device(d.data_ptr(), b.shape[0])
        assert np.array_equal(e.inliers, eb.inliers) and np.array_equal(e.rotation, eb.rotation)
    # a graph captured before a reallocation is never replayed again, even after the key's next
    # eager run re-arms it (regression: the staged small-input path hit exactly this)
    e_a = runs[0]
    ctx.estimate_single_device(db.data_ptr(), big.shape[0])  # grow again between the eager runs
    for data, want in ((a, e_a), (b, eb), (a, e_a)):
        d.copy_(torch.from_numpy(data))
        for _ in range(2):
            e = ctx.estimate_single_device(d.data_ptr(), data.shape[0])
            assert np.array_equal(e.inliers, want.inliers) and np.array_equal(e.rotation, want.rotation)
    small = [synth.make_scene(200, 0.2, 0.01, seed=229 + k)[0] for k in range(4)]
    want_small = [port.estimate_single(x) for x in small]
    for rep in range(3):  # staged pageable small inputs: eager, capture, replays
        for x, w in zip(small, want_small):
            assert_est_equal(ctx.estimate_single(x), w)
        ctx.estimate_single(big[:300_000])  # a different solve in between (buffer growth on rep 0)


@pytest.mark.parametrize("world", [2, 8])
def test_sharded_vote_protocol_single_gpu(ctx, world):
    # the multi-GPU protocol emulated sequentially on one GPU (no cross-kernel waits): per-shard
    # votes summed (what the NCCL all-reduce does) + finish on the gathered input must equal the
    # single solve bit-for-bit
    import torch
    from paper_2502_06337_b200 import distributed as rvd
    corrs, _, _ = synth.make_config("c3", 300_000)
    d = torch.from_numpy(corrs).cuda()
    # the context runs on torch's stream: `total += g` is ordered before the C-ABI calls
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    total = torch.zeros((512, 512), dtype=torch.int32, device="cuda")
    for r in range(world):
        lo, hi = rvd.shard_bounds(corrs.shape[0], world, r)
        g = torch.empty((512, 512), dtype=torch.int32, device="cuda")
        ctx.vote_shard(d[lo:hi].data_ptr(), hi - lo, g.data_ptr())
        total += g
    e = ctx.estimate_single_prevoted(d.data_ptr(), corrs.shape[0], total.data_ptr())
    z, _, _ = ctx.preprocess(corrs)
    ref_grid = ctx.accumulate(z)
    assert np.array_equal(total.cpu().numpy().view(np.uint32), ref_grid)
    assert ctx.stage_times()["vote_guard_reruns"] == 0  # the prevoted grid was used, not re-voted
    e1 = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0])
    assert np.array_equal(e.inliers, e1.inliers) and np.array_equal(e.rotation, e1.rotation)
    ctx.set_stream(None)


def test_full_size_multi_recovers_three(ctx):
    corrs, rots, _ = synth.make_config("c5")
    ms = ctx.estimate_multi(corrs, rv.EstimatorConfig(max_models=3))
    assert len(ms) == 3
    errs = [min(orc.rotation_error_deg(r, m.rotation) for m in ms) for r in rots]
    assert max(errs) < 0.1


# ---- one-pass top-K multi-model mode (an extension: no reference twin) ----
@pytest.mark.gpu
def test_multi_onepass_recovers_the_sequential_models(ctx, port):
    corrs, rots, _ = synth.make_config("c5", 50_000)
    cfg = rv.EstimatorConfig(max_models=3)
    seq = port.estimate_multi(corrs, orc.default_config(max_models=3))
    one = ctx.estimate_multi_onepass(corrs, cfg)
    assert len(one) == len(seq) == 3
    assert [m.axis_votes for m in one] == sorted([m.axis_votes for m in one], reverse=True)
    for r in rots:  # every ground-truth rotation is found by both modes to the same accuracy class
        e_one = min(orc.rotation_error_deg(r, m.rotation) for m in one)
        e_seq = min(orc.rotation_error_deg(r, m["rotation"]) for m in seq)
        assert e_one < 0.5 and e_seq < 0.5
    # the first (strongest) model is the same peak as the sequential first round
    assert one[0].axis_votes == seq[0]["axis_votes"]
    assert np.array_equal(one[0].inliers, seq[0]["inliers"])


# ---- batched solver for independent problems (an extension) ----------
def test_estimate_batch_matches_single_solves(ctx, port):
    rng = np.random.default_rng(7)
    probs = []
    for k in range(24):
        n = int(rng.integers(300, 6000))
        corrs, _, _ = synth.make_scene(n, 0.6, 0.01, seed=9000 + k)
        probs.append(corrs)
    probs.append(np.zeros((0, 6)))                      # an empty problem fails alone
    res = ctx.estimate_batch(probs, workers=6)
    assert len(res) == len(probs)
    assert isinstance(res[-1], rv.errors.EmptyInput)
    for k, corrs in enumerate(probs[:-1]):
        ref = port.estimate_single(corrs)
        assert_est_equal(res[k], ref)


# ---- baseline consensus kernels vs the compiled reference -----------
def test_grid_oracle_axis_matches_reference(ctx, ref):
    corrs, _, _ = synth.make_config("c2", 20_000)
    z, _, _ = ref.preprocess(corrs)
    ax_r, cnt_r = ref.grid_oracle_axis(z, 2000, 0.015)
    ax_d, cnt_d = ctx.grid_oracle_axis(z, 2000, 0.015)
    assert cnt_d == cnt_r and np.array_equal(ax_d, ax_r)


def test_consensus_counts_exact_at_band_edges(ctx, ref):
    rng = np.random.default_rng(3)
    z = unit_rows(rng, 5000)
    axes = unit_rows(rng, 300)
    # constraints placed exactly at |a.z| = eps +- 1 ulp-ish for the first axis
    a0 = axes[0]
    t = np.cross(a0, [0.0, 0.0, 1.0])
    t /= np.linalg.norm(t)
    edge = np.array([np.cos(np.arcsin(e)) * t + e * a0 for e in (0.015, 0.015 - 1e-12, 0.015 + 1e-12, -0.015)])
    z = np.concatenate([z, edge])
    got = ctx.consensus_counts(axes, z, 0.015)
    want = np.array([len(ref.classify_inliers(a, z, 0.015)) for a in axes], np.uint32)
    assert np.array_equal(got, want)


@pytest.mark.parametrize("seed", [0, 7])
def test_ransac_rotation_matches_reference(ctx, ref, seed):
    corrs, _, _ = synth.make_config("c1")
    r = ref.ransac_rotation(corrs, 300, 0.015, seed)
    d = ctx.ransac_rotation(corrs, 300, 0.015, seed)
    assert d.axis_votes == r["axis_votes"]
    assert np.array_equal(d.inliers, r["inliers"])
    assert orc.rotation_error_deg(d.rotation, r["rotation"]) <= ROT_TOL_DEG

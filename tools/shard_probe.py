"""Dev probe: per-rank pieces of the sharded solve (distributed.py / rv_multi)
timed on one GPU for P ranks, C3 (N = 1e6): the shard vote (N/P rows, CUDA events), and the
sharded finish steps of one rank (peak + start axis from the summed grid, one classify pass of its
shard, its angle histogram and window sums; each is a synchronous C-ABI call, timed on the host
including the call overhead). Also the full rv_multi solve at P = 1 (the real NCCL clique)."""
import json
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402


def host_ms(fn, reps=10):
    ts = []
    for _ in range(reps + 3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        ts.append(1e3 * (time.perf_counter() - t0))
    return statistics.median(ts[3:])


corrs, _, _ = synth.make_config("c3")
n = corrs.shape[0]
ctx = rv.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
cfg = rv.EstimatorConfig()
d = torch.from_numpy(corrs).cuda()
grid = torch.zeros((cfg.grid, cfg.grid), dtype=torch.int32, device="cuda")
ctx.vote_shard(d.data_ptr(), n, grid.data_ptr(), cfg)  # full grid (= the all-reduced one)
axis, votes, total = ctx.peak_start_axis(grid.data_ptr(), cfg)
rows = []
for P in (1, 2, 4, 8):
    lo, hi = 0, n // P
    shard = d[lo:hi]
    g = torch.zeros_like(grid)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    tv = []
    for it in range(10):
        ev[0].record()
        ctx.vote_shard(shard.data_ptr(), hi - lo, g.data_ptr(), cfg)
        ev[1].record()
        torch.cuda.synchronize()
        if it >= 3:
            tv.append(ev[0].elapsed_time(ev[1]))
    # this context now holds the shard: the finish steps of one rank
    t_peak = host_ms(lambda: ctx.peak_start_axis(grid.data_ptr(), cfg))
    t_cls = host_ms(lambda: ctx.shard_classify(axis, cfg.epsilon, 0, False))
    bins, _ = ctx.shard_angle_hist(axis, cfg)
    t_ang = host_ms(lambda: ctx.shard_angle_hist(axis, cfg))
    t_sum = host_ms(lambda: ctx.shard_angle_sums(bins, cfg))
    row = {"P": P, "shard_rows": hi - lo, "shard_vote_ms": statistics.median(tv), "peak_start_axis_ms": t_peak,
           "classify_pass_ms": t_cls, "angle_hist_ms": t_ang, "angle_sums_ms": t_sum}
    rows.append(row)
    print(json.dumps(row), flush=True)
m = rv.MultiContext([0])
m.estimate_single(corrs, cfg)
t_multi = host_ms(lambda: m.estimate_single(corrs, cfg), reps=5)
print(json.dumps({"rv_multi_P1_estimate_single_ms": t_multi, "nccl_version": m.nccl_version}))

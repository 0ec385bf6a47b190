"""Dev probe: per-rank pieces of the sharded solve (distributed.py) timed on one GPU for P ranks:
the shard vote (N/P rows) and the replicated finish from the reduced grid (N rows)."""
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

corrs, _, _ = synth.make_config("c3")
n = corrs.shape[0]
ctx = rv.Context(0)
cfg = rv.EstimatorConfig()
d = torch.from_numpy(corrs).cuda()
grid = torch.zeros((cfg.grid, cfg.grid), dtype=torch.int32, device="cuda")
ctx.vote_shard(d.data_ptr(), n, grid.data_ptr(), cfg)  # full grid (= the all-reduced one)
for P in (2, 4, 8):
    lo, hi = 0, n // P
    shard = d[lo:hi]
    g = torch.zeros_like(grid)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tv, tf = [], []
    for it in range(8):
        ev[0].record()
        ctx.vote_shard(shard.data_ptr(), hi - lo, g.data_ptr(), cfg)
        ev[1].record()
        ctx.estimate_single_prevoted(d.data_ptr(), n, grid.data_ptr(), cfg)
        ev[2].record()
        torch.cuda.synchronize()
        if it >= 3:
            tv.append(ev[0].elapsed_time(ev[1]))
            tf.append(ev[1].elapsed_time(ev[2]))
    print(f"P={P}: shard vote {np.median(tv):.3f} ms, replicated finish {np.median(tf):.3f} ms")

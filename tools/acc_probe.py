"""Dev probe: accumulate (vote only) timing per config size, stage timers on, median of reps."""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

ctx = rv.Context(0)
ctx.enable_timing(True)
for key, n in (("c1", 1000), ("c2", 100_000), ("c3", 1_000_000)):
    corrs, _, _ = synth.make_config(key, n)
    z, _, _ = ctx.preprocess(corrs)
    t = []
    for _ in range(7):
        ctx.accumulate(z)
        t.append(ctx.stage_times()["vote_ms"])
    print(key, n, "vote_ms median", round(float(np.median(t[2:])), 3), [round(x, 3) for x in t])

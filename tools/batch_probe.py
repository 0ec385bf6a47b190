"""Dev probe: throughput of the batched solver vs one-at-a-time solves (independent problems)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

ctx = rv.Context(0)
for n, B in ((1000, 256), (10000, 128), (100000, 16)):
    probs = [synth.make_scene(n, 0.9, 0.01, seed=100 + k)[0] for k in range(B)]
    ctx.estimate_batch(probs[:4])
    t0 = time.perf_counter()
    for p in probs:
        ctx.estimate_single(p)
    t1 = time.perf_counter()
    for w in (4, 8, 16):
        ctx.estimate_batch(probs[:3 * w], workers=w)  # warm: allocations + graph capture per worker
        t2 = time.perf_counter()
        res = ctx.estimate_batch(probs, workers=w)
        t3 = time.perf_counter()
        print(f"n={n} B={B}: sequential {1e3 * (t1 - t0) / B:.3f} ms/problem, batch(workers={w}) "
              f"{1e3 * (t3 - t2) / B:.3f} ms/problem -> {(t1 - t0) / (t3 - t2):.1f}x, "
              f"{n * B / (t3 - t2):.3e} corr/s", flush=True)

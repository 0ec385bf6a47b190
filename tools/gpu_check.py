"""Ad-hoc GPU parity/timing probe used during development (not part of the test suite)."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402

import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402


def main():
    port = orc.Oracle("port")
    ctx = rv.Context(0)
    ctx.enable_timing(True)
    for key, n in [("c1", None), ("c2", 100_000), ("c4", 50_000), ("c5", 50_000)]:
        corrs, rots, _ = synth.make_config(key, n)
        z, kept, _ = port.preprocess(corrs)
        t0 = time.time()
        g_ref = port.accumulate(z)
        t1 = time.time()
        g_dev = ctx.accumulate(z)
        st = ctx.stage_times()
        bad = int((g_dev != g_ref).sum())
        print(f"{key} n={len(z)} grid mismatch cells={bad} sum dev={int(g_dev.sum(dtype=np.uint64))} "
              f"ref={int(g_ref.sum(dtype=np.uint64))} oracle {t1 - t0:.2f}s vote {st['vote_ms']:.3f} ms "
              f"pairs={st['vote_pairs']} samples={st['vote_samples']}", flush=True)
        if bad:
            idx = np.argwhere(g_dev != g_ref)[:5]
            for iy, ix in idx:
                print("   cell", iy, ix, g_dev[iy, ix], g_ref[iy, ix])
    for key, n in [("c1", None), ("c2", 100_000), ("c4", 100_000)]:
        corrs, rots, _ = synth.make_config(key, n)
        e = ctx.estimate_single(corrs)
        st = ctx.stage_times()
        r = port.estimate_single(corrs)
        print(f"{key} estimate: inliers equal={np.array_equal(e.inliers, r['inliers'])} ({e.inliers.size} vs "
              f"{r['inliers'].size}) rotdiff={orc.rotation_error_deg(e.rotation, r['rotation']):.2e} deg "
              f"votes {e.axis_votes}/{r['axis_votes']} trace={port.trace()} times={st}", flush=True)
    corrs, rots, _ = synth.make_config("c5", 50_000)
    cfg = rv.EstimatorConfig(max_models=3)
    ms = ctx.estimate_multi(corrs, cfg)
    rs = port.estimate_multi(corrs, orc.default_config(max_models=3))
    print("c5 multi", len(ms), len(rs),
          [(np.array_equal(a.inliers, b["inliers"]), orc.rotation_error_deg(a.rotation, b["rotation"])) for a, b in
           zip(ms, rs)], flush=True)
    for key in ["c3", "c4", "c5"]:
        corrs, rots, _ = synth.make_config(key)
        cfg = rv.EstimatorConfig(max_models=3 if key == "c5" else 1)
        import torch
        d = torch.from_numpy(corrs).cuda()
        torch.cuda.synchronize()
        for rep in range(3):
            t0 = time.time()
            if key == "c5":
                ms = ctx.estimate_multi_device(d.data_ptr(), corrs.shape[0], cfg)
                e = ms[0]
            else:
                e = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
            t1 = time.time()
        st = ctx.stage_times()
        print(f"{key} full device solve {1e3 * (t1 - t0):.2f} ms wall, err vs truth "
              f"{orc.rotation_error_deg(rots[0], e.rotation):.4f} deg, inliers {e.inliers.size}, times {st}",
              flush=True)


if __name__ == "__main__":
    main()

"""C1-C5 measurement table (BASELINE.md "GPU measurement"): one B200, one run of this script.

Per BASELINE config at its full size:
  device   ms per solve with the input resident in HBM (median of the timed reps, CUDA events
           around the call; estimate_single for C1-C4, estimate_multi(max_models=3) for C5)
  e2e      the same through the host-input C-ABI from pinned memory (H2D inside)
  pageable the same from a pageable numpy array (the C++ drop-in's path)
  vote     the band-tiled vote kernel's own time and its fraction of the measured smem-atomic peak
  cpu      the reference (oracle/_ref, -O3 -march=native) at cfg.threads = 1 and = nproc, bounded
           runs (1 rep for the 1e6 configs at 1 thread)
Writes a JSON document on stdout and a markdown table on stderr.
"""
import json
import os
import statistics
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402

import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

sys.path.insert(0, str(ROOT))
import bench  # noqa: E402


def timed(fn, reps):
    ms = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ms.append(max(a.elapsed_time(b), 1e3 * (time.perf_counter() - t0)))
    return statistics.median(ms)


def main():
    ctx = rv.Context(0)
    ctx.set_stream(torch.cuda.current_stream().cuda_stream)
    peak = bench.smem_atomic_peak(0)
    nproc = os.cpu_count() or 1
    ref = orc.Oracle("ref_perf")
    rows = []
    for key in ("c1", "c2", "c3", "c4", "c5"):
        corrs, rots, _ = synth.make_config(key)
        n = corrs.shape[0]
        multi = key == "c5"
        cfg = rv.EstimatorConfig(max_models=3 if multi else 1)
        d = torch.from_numpy(corrs).cuda()
        pinned = torch.empty((n, 6), dtype=torch.float64, pin_memory=True)
        pinned.numpy()[:] = corrs
        reps = 20 if n <= 100_000 else 10
        if multi:
            dev = lambda: ctx.estimate_multi_device(d.data_ptr(), n, cfg)  # noqa: E731
            e2e = lambda: ctx.estimate_multi(pinned.numpy(), cfg)  # noqa: E731
            pag = lambda: ctx.estimate_multi(corrs, cfg)  # noqa: E731
        else:
            dev = lambda: ctx.estimate_single_device(d.data_ptr(), n, cfg)  # noqa: E731
            e2e = lambda: ctx.estimate_single(pinned.numpy(), cfg)  # noqa: E731
            pag = lambda: ctx.estimate_single(corrs, cfg)  # noqa: E731
        for f in (dev, e2e, pag):
            f()
            f()
        t_dev, t_e2e, t_pag = timed(dev, reps), timed(e2e, reps), timed(pag, reps)
        ctx.enable_timing(True)
        dev()
        st = ctx.stage_times()
        ctx.enable_timing(False)
        vote_ms = st["vote_kernel_ms"] / max(1, st["vote_launches"])
        frac = (st["vote_samples"] / max(1, st["vote_launches"])) / (vote_ms * 1e-3) / peak if peak and vote_ms else None
        ocfg = orc.default_config(max_models=3) if multi else orc.default_config()
        cpu = {}
        for threads in (1, nproc):
            ocfg.threads = threads
            k = 1 if (n >= 1_000_000 and threads == 1) else 3
            ts = []
            for _ in range(k):
                t0 = time.perf_counter()
                (ref.estimate_multi if multi else ref.estimate_single)(corrs, ocfg)
                ts.append(time.perf_counter() - t0)
            cpu[threads] = 1e3 * statistics.median(ts)
        row = {"config": key, "n": n, "call": "estimate_multi(K=3)" if multi else "estimate_single",
               "device_ms": t_dev, "e2e_pinned_ms": t_e2e, "e2e_pageable_ms": t_pag,
               "corr_per_s": n / (t_dev * 1e-3), "vote_kernel_ms": vote_ms, "vote_launches": st["vote_launches"],
               "vote_frac_smem_atomic": frac, "cpu_1thread_ms": cpu[1], "cpu_nproc_ms": cpu[nproc], "nproc": nproc,
               "speedup_e2e_vs_cpu_nproc": cpu[nproc] / t_e2e}
        rows.append(row)
        print(json.dumps(row), file=sys.stderr, flush=True)
    print(json.dumps({"rows": rows, "gpu": torch.cuda.get_device_name(0), "smem_atomic_peak": peak}))
    hdr = ("| Config | call | N | device ms | e2e pinned ms | e2e pageable ms | corr/s (device) | vote kernel ms "
           "| vote frac | CPU 1-thread ms | CPU %d-thread ms |" % nproc)
    print("\n" + hdr, file=sys.stderr)
    print("|" + "---|" * 11, file=sys.stderr)
    for r in rows:
        print(f"| {r['config'].upper()} | {r['call']} | {r['n']:,} | {r['device_ms']:.3f} | {r['e2e_pinned_ms']:.3f} | "
              f"{r['e2e_pageable_ms']:.3f} | {r['corr_per_s']:.3g} | {r['vote_kernel_ms']:.3f} "
              f"(x{r['vote_launches']}) | {r['vote_frac_smem_atomic'] or 0:.3f} | {r['cpu_1thread_ms']:.1f} | "
              f"{r['cpu_nproc_ms']:.1f} |", file=sys.stderr)


if __name__ == "__main__":
    main()

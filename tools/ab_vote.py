"""Dev A/B of vote-kernel variants on one B200: each argument is a library built by
`RV_NVCC_EXTRA=... RV_LIB_OUT=_variants/<name> python paper_2502_06337_b200/build.py --force`.
Runs C3 (AB_CONFIG) device solves with per-stage timers in a fresh process per (variant, round), variants
interleaved over rounds; prints the median vote-kernel time and device solve time per variant."""
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import os, sys, json, torch
sys.path.insert(0, %r)
import paper_2502_06337_b200 as rv
from paper_2502_06337_b200 import synth
corrs, _, _ = synth.make_config(os.environ.get("AB_CONFIG", "c3"))
ctx = rv.Context(0)
d = torch.from_numpy(corrs).cuda()
cfg = rv.EstimatorConfig()
flush = torch.empty(64 << 20, dtype=torch.int32, device="cuda")
for _ in range(3):
    ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
ctx.enable_timing(True)
vk, vs = [], []
for _ in range(15):
    flush.zero_()
    ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
    st = ctx.stage_times()
    vk.append(st["vote_kernel_ms"]); vs.append(st["total_ms"])
ctx.enable_timing(False)
# end to end from pinned host memory (the pipelined chunked path), CUDA events on the current stream
h = torch.empty((corrs.shape[0], 6), dtype=torch.float64, pin_memory=True)
h.numpy()[:] = corrs
for _ in range(3):
    ctx.estimate_single(h.numpy(), cfg)
e2e = []
for _ in range(15):
    flush.zero_()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    ctx.estimate_single(h.numpy(), cfg)
    b.record()
    torch.cuda.synchronize()
    e2e.append(a.elapsed_time(b))
print(json.dumps({"vote_kernel_ms": vk, "total_ms": vs, "e2e_ms": e2e}))
"""
libs = sys.argv[1:]
rounds = int(os.environ.get("AB_ROUNDS", "3"))
res = {l: {"vote_kernel_ms": [], "total_ms": [], "e2e_ms": []} for l in libs}
for r in range(rounds):
    for l in libs:
        # "dir" or "dir@VAR=value@VAR2=value2": a variant library plus run-time knobs
        parts = l.split("@")
        env = dict(os.environ, RV_LIB_PATH=str(Path(parts[0]) / "librotavote_b200.so"))
        env.update(kv.split("=", 1) for kv in parts[1:])
        out = subprocess.run([sys.executable, "-c", CHILD % str(ROOT)], env=env, capture_output=True, text=True)
        if out.returncode != 0:
            print(l, "FAILED", out.stderr[-2000:])
            continue
        d = json.loads(out.stdout.strip().splitlines()[-1])
        for k in d:
            res[l][k] += d[k]
for l in libs:
    v = res[l]
    if v["vote_kernel_ms"]:
        print(f"{l:40s} vote_kernel {statistics.median(v['vote_kernel_ms']):.4f} ms  stages {statistics.median(v['total_ms']):.4f} ms  "
              f"e2e {statistics.median(v['e2e_ms']):.4f} ms  (n={len(v['vote_kernel_ms'])})")

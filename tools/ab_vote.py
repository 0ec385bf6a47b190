"""Dev A/B of vote-kernel variants on one B200: each argument is a library built by
`RV_NVCC_EXTRA=... RV_LIB_OUT=_variants/<name> python paper_2502_06337_b200/build.py --force`.
Runs C3 device solves with per-stage timers in a fresh process per (variant, round), variants
interleaved over rounds; prints the median vote-kernel time and device solve time per variant."""
import json
import os
import statistics
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import sys, json, torch
sys.path.insert(0, %r)
import paper_2502_06337_b200 as rv
from paper_2502_06337_b200 import synth
corrs, _, _ = synth.make_config("c3")
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
print(json.dumps({"vote_kernel_ms": vk, "total_ms": vs}))
"""
libs = sys.argv[1:]
rounds = int(os.environ.get("AB_ROUNDS", "3"))
res = {l: {"vote_kernel_ms": [], "total_ms": []} for l in libs}
for r in range(rounds):
    for l in libs:
        env = dict(os.environ, RV_LIB_PATH=str(Path(l) / "librotavote_b200.so"))
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
        print(f"{l:40s} vote_kernel {statistics.median(v['vote_kernel_ms']):.4f} ms  stages {statistics.median(v['total_ms']):.4f} ms  (n={len(v['vote_kernel_ms'])})")

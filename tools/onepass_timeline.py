"""Dev probe: device timeline of one C5 one-pass multi-model solve (torch.profiler)."""
import json
import sys
import tempfile
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

corrs, _, _ = synth.make_config("c5")
ctx = rv.Context(0)
d = torch.from_numpy(corrs).cuda()
cfg = rv.EstimatorConfig(max_models=3)
mode = sys.argv[1] if len(sys.argv) > 1 else "onepass"
fn = (lambda: ctx.estimate_multi_onepass_device(d.data_ptr(), corrs.shape[0], cfg)) if mode == "onepass" else \
    (lambda: ctx.estimate_multi_device(d.data_ptr(), corrs.shape[0], cfg))
for _ in range(2):
    fn()
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    fn()
    torch.cuda.synchronize()
with tempfile.NamedTemporaryFile(suffix=".json") as f:
    prof.export_chrome_trace(f.name)
    ev = json.load(open(f.name))["traceEvents"]
acts = sorted([e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memset", "gpu_memcpy")],
              key=lambda e: e["ts"])
t0 = acts[0]["ts"]
agg = {}
end_prev = t0
idle = 0.0
for e in acts:
    idle += max(0.0, e["ts"] - end_prev)
    end_prev = max(end_prev, e["ts"] + e["dur"])
    nm = e["name"]
    k = nm.split("::")[-1].split("(")[0] if "::" in nm else nm[:40]
    k = k.split("<")[0] if k.startswith(("vote", "plan", "preprocess")) else k
    a = agg.setdefault(k, [0, 0.0])
    a[0] += 1
    a[1] += e["dur"]
print(f"span {end_prev - t0:.1f} us, idle {idle:.1f} us, {len(acts)} activities")
if "seq" in sys.argv[2:]:
    prev = t0
    for e in acts:
        print(f"{e['ts'] - t0:8.1f} gap {e['ts'] - prev:7.1f} dur {e['dur']:8.1f} {e['name'][:60]}")
        prev = e["ts"] + e["dur"]
for k, (cnt, tot) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:15]:
    print(f"{cnt:4d} x  {tot:9.1f} us  {k}")

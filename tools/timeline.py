"""Dev probe: device timeline of one C3 solve via torch.profiler (CUPTI activity records of every
kernel / memset / memcpy in the process, including the library's own launches). Prints each
activity with its start offset, duration and the idle gap before it."""
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

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
host = "host" in sys.argv[2:]
flush_l2 = "flush" in sys.argv[2:]  # like bench.py: 256 MiB write + sync before the solve
show_api = "api" in sys.argv[2:]  # also list the host-side CUDA runtime calls
corrs, _, _ = synth.make_config(key)
ctx = rv.Context(0)
ctx.set_stream(torch.cuda.current_stream().cuda_stream)
d = torch.from_numpy(corrs).cuda()
h = torch.empty((corrs.shape[0], 6), dtype=torch.float64, pin_memory=True)
h.numpy()[:] = corrs
cfg = rv.EstimatorConfig()


multi = "multi" in sys.argv[2:]  # estimate_multi (max_models=3)
if multi:
    cfg = rv.EstimatorConfig(max_models=3)


def solve():
    if multi:
        return ctx.estimate_multi_device(d.data_ptr(), corrs.shape[0], cfg)
    if host:
        return ctx.estimate_single(h.numpy(), cfg)
    return ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)


flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for _ in range(3):
    solve()
torch.cuda.synchronize()
if flush_l2:
    flush.zero_()
    torch.cuda.synchronize()
acts_kind = [ProfilerActivity.CUDA] + ([ProfilerActivity.CPU] if show_api else [])
with profile(activities=acts_kind) as prof:
    solve()
    torch.cuda.synchronize()
with tempfile.NamedTemporaryFile(suffix=".json") as f:
    prof.export_chrome_trace(f.name)
    ev = json.load(open(f.name))["traceEvents"]
cats = ("kernel", "gpu_memset", "gpu_memcpy") + (("cuda_runtime", "cuda_driver") if show_api else ())
acts = [e for e in ev if e.get("ph") == "X" and e.get("cat") in cats]
acts.sort(key=lambda e: e["ts"])
t0 = acts[0]["ts"]
end_prev = t0
busy = 0.0
for e in acts:
    gap = e["ts"] - end_prev
    print(f"{e['ts'] - t0:9.1f} us  dur {e['dur']:8.1f}  gap {gap:7.1f}  {e['cat']:10s} {e['name'][:70]}")
    if e["cat"] in ("cuda_runtime", "cuda_driver"):
        continue
    end_prev = max(end_prev, e["ts"] + e["dur"])
    busy += e["dur"]
span = end_prev - t0
print(f"span {span:.1f} us, busy {busy:.1f} us, idle {span - busy:.1f} us")

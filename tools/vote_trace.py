"""Dev probe (needs a build with RV_NVCC_EXTRA=-DRV_VOTE_TRACE): per-CTA phase timeline of the
banded vote launches of one C3 solve (device-resident, then host input): init, band visits,
flushes and the launch tail."""
import ctypes as C
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

corrs, _, _ = synth.make_config(sys.argv[1] if len(sys.argv) > 1 else "c3")
ctx = rv.Context(0)
d = torch.from_numpy(corrs).cuda()
h = torch.empty((corrs.shape[0], 6), dtype=torch.float64, pin_memory=True)
h.numpy()[:] = corrs
from paper_2502_06337_b200 import _native  # noqa: E402

lib = C.CDLL(str(_native.LIB_PATH))  # the library the context uses (RV_LIB_PATH for variants)
buf = (C.c_ulonglong * (2 * 65536))()


def analyse(label):
    n = lib.rv_debug_vote_trace(buf, 65536)
    a = np.frombuffer(buf, dtype=np.uint64, count=2 * n).reshape(-1, 2)
    per = defaultdict(list)
    for t, info in a:
        per[int(info) >> 16].append((int(t), (int(info) >> 8) & 255, int(info) & 255))
    launches = defaultdict(dict)  # launch index -> cta -> events
    for cta, ev in per.items():
        ev.sort()
        k = -1
        for e in ev:
            if e[1] == 0:
                k += 1
                launches[k][cta] = []
            launches[k][cta].append(e)
    for k in sorted(launches):
        L = launches[k]
        t0 = min(ev[0][0] for ev in L.values())
        ends = np.array([ev[-1][0] - t0 for ev in L.values()]) / 1e3
        starts = np.array([ev[0][0] - t0 for ev in L.values()]) / 1e3
        init = np.array([ev[1][0] - ev[0][0] for ev in L.values()]) / 1e3
        visits = np.array([sum(1 for e in ev if e[1] == 2) for ev in L.values()])
        flush = np.array([sum(e3[0] - e2[0] for e2, e3 in zip(ev, ev[1:]) if e2[1] == 2 and e3[1] == 3)
                          for ev in L.values()]) / 1e3
        zero = np.array([sum(e2[0] - e3[0] for e3, e2 in zip(ev, ev[1:]) if e3[1] == 3 and e2[1] == 2)
                         for ev in L.values()]) / 1e3  # zero + the next visit's votes (upper bound)
        slow = max(L.values(), key=lambda ev: ev[-1][0])
        t_s = slow[0][0]
        print(f"  slowest cta: " + " ".join(f"tag{e[1]}@{(e[0] - t_s) / 1e3:.1f}(b{e[2]})" for e in slow))
        print(f"{label} launch {k}: ctas={len(L)} span={ends.max():.1f}us start max={starts.max():.1f} "
              f"init med={np.median(init):.1f} end min/med/max={ends.min():.1f}/{np.median(ends):.1f}/{ends.max():.1f} "
              f"visits mean={visits.mean():.2f} max={visits.max()} flush/cta med={np.median(flush):.1f}us "
              f"idle-tail sum={np.sum(ends.max() - ends):.0f} cta-us ({np.mean(ends.max() - ends) / ends.max():.1%})")


cfg = rv.EstimatorConfig()
for _ in range(2):
    ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
    ctx.estimate_single(h.numpy(), cfg)
torch.cuda.synchronize()
lib.rv_debug_vote_trace(buf, 65536)
ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
torch.cuda.synchronize()
analyse("device")
ctx.estimate_single(h.numpy(), cfg)
torch.cuda.synchronize()
analyse("host")

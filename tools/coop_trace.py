"""Dev probe (needs a build with RV_NVCC_EXTRA=-DRV_COOP_TRACE): per-phase timings of the
cooperative refine kernel's passes on a C4 solve."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c4"
corrs, _, _ = synth.make_config(key)
ctx = rv.Context(0)
d = torch.from_numpy(corrs).cuda()
lib = C.CDLL(str(ROOT / "paper_2502_06337_b200" / "_lib" / "librotavote_b200.so"))
buf = (C.c_ulonglong * 8192)()
for rep in range(2):
    lib.rv_debug_coop_trace(buf, 8192)
    ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], rv.EstimatorConfig())
    torch.cuda.synchronize()
n = lib.rv_debug_coop_trace(buf, 8192)
ev = [(int(x) >> 4, int(x) & 15) for x in buf[:n]]
ph = {1: [], 2: [], 3: [], 4: [], 5: [], 6: [], 7: [], 8: []}
passes = 0
for k in range(1, len(ev)):
    t, tag = ev[k]
    tp, tagp = ev[k - 1]
    if tag in (2, 3, 4, 5, 6, 8) and tagp == tag - 1:
        ph[tag].append(t - tp)
    if tag == 1 and tagp == 6:
        ph[1].append(t - tp)
    if tag == 1:
        passes += 1
names = {2: "classify", 3: "block reduce", 4: "barrier", 5: "partials reduce", 6: "decision", 1: "loop",
         8: "final flags+compaction"}
print(f"passes={passes}")
tail = [(t, tag) for t, tag in ev if tag in (6, 7, 8, 9, 10)]
print("last events:", [(tag, round((t - tail[-6][0]) / 1e3, 2)) for t, tag in tail[-6:]])
for tag in (2, 3, 4, 5, 6, 1, 8):
    if ph[tag]:
        a = np.array(ph[tag]) / 1e3
        print(f"{names[tag]:>16}: mean {a.mean():7.2f} us  median {np.median(a):7.2f}  max {a.max():7.2f}  n={a.size}")

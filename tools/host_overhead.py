"""Dev probe: where the host time of one device-resident C3 solve goes (Python wrapper, C call,
result copy) next to the CUDA-event device span."""
import ctypes as C
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402
from paper_2502_06337_b200._native import rv_estimate  # noqa: E402

corrs, _, _ = synth.make_config("c3")
ctx = rv.Context(0)
st = torch.cuda.current_stream()
ctx.set_stream(st.cuda_stream)
d = torch.from_numpy(corrs).cuda()
cfg = rv.EstimatorConfig()
c = cfg.to_c()
for _ in range(5):
    ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
torch.cuda.synchronize()
R = 20
t_call, t_res, t_tot, t_ev = [], [], [], []
e = rv_estimate()
inl = np.empty(corrs.shape[0], np.int32)
for _ in range(R):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(st)
    ctx._lib.rv_estimate_single_device(ctx.handle, C.c_void_p(d.data_ptr()), corrs.shape[0], C.byref(c), C.byref(e))
    t1 = time.perf_counter()
    ctx._lib.rv_result_inliers(ctx.handle, 0, inl.ctypes.data_as(C.POINTER(C.c_int32)), int(e.n_inliers))
    t2 = time.perf_counter()
    b.record(st)
    torch.cuda.synchronize()
    t_call.append(t1 - t0); t_res.append(t2 - t1); t_ev.append(a.elapsed_time(b))
for _ in range(R):
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.record(st)
    ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], cfg)
    b.record(st)
    torch.cuda.synchronize()
    t_tot.append((time.perf_counter() - t0, a.elapsed_time(b)))
m = lambda v: 1e3 * float(np.median(v))
print(f"raw C call {m(t_call):.3f} ms, rv_result_inliers {m(t_res):.3f} ms, events {float(np.median(t_ev)):.3f} ms")
print(f"python API wall {m([x[0] for x in t_tot]):.3f} ms, events {float(np.median([x[1] for x in t_tot])):.3f} ms")

"""CSV ingest measurement: a C3-sized correspondence file in the
reference writer's format (header + %.17g, io.cpp:103-110), parsed by
  * the reference's read_correspondences (oracle/_ref perf build, one host thread: io.cpp is serial),
  * rv_read_correspondences_csv (file read into pinned memory + H2D + device parse),
  * rv_parse_correspondences_csv from text already in pinned host memory,
and the device kernels alone (CUDA events around the parse of device-resident... text staged by
the call). Prints one JSON line."""
import ctypes as C
import json
import os
import sys
import tempfile
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
corrs, _, _ = synth.make_config("c3", n)
text = ("x0,x1,x2,y0,y1,y2\n" + "\n".join(",".join("%.17g" % v for v in row) for row in corrs) + "\n").encode()
path = Path(tempfile.gettempdir()) / f"rv_io_bench_{n}.csv"
path.write_bytes(text)
mb = len(text) / 1e6

ctx = rv.Context(0)
for _ in range(2):
    d, m = ctx.read_correspondences_device(str(path))
torch.cuda.synchronize()
reps = 10
t = []
for _ in range(reps):
    t0 = time.perf_counter()
    d, m = ctx.read_correspondences_device(str(path))
    t.append(time.perf_counter() - t0)
t_file = float(np.median(t))

pinned = torch.empty(len(text), dtype=torch.uint8, pin_memory=True)
pinned.numpy()[:] = np.frombuffer(text, np.uint8)
ptr = C.c_char_p(pinned.data_ptr())
dp, nr, ln = C.c_void_p(), C.c_int64(), C.c_int64()
lib = ctx._lib
lib.rv_parse_correspondences_csv.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(C.c_void_p),
                                             C.POINTER(C.c_int64), C.POINTER(C.c_int64)]
t = []
ctx.enable_timing(True)
kern = []
for _ in range(reps):
    t0 = time.perf_counter()
    st = lib.rv_parse_correspondences_csv(ctx.handle, C.c_void_p(pinned.data_ptr()), len(text), C.byref(dp),
                                          C.byref(nr), C.byref(ln))
    t.append(time.perf_counter() - t0)
    assert st == 0
    kern.append(ctx.stage_times()["preprocess_ms"])
ctx.enable_timing(False)
t_mem = float(np.median(t))
got = ctx._rows_to_host(dp.value, nr.value)
assert np.array_equal(got.view(np.uint64), corrs.view(np.uint64))

import oracle as orc  # noqa: E402
ref = orc.Oracle("ref_perf")
t = []
for _ in range(3):
    t0 = time.perf_counter()
    rows, err = ref.read_correspondences(path)
    t.append(time.perf_counter() - t0)
assert err is None and np.array_equal(rows.view(np.uint64), corrs.view(np.uint64))
t_ref = float(np.median(t))
hbm = 6456.5
k_ms = float(np.median(kern))
print(json.dumps({
    "rows": n, "text_MB": round(mb, 1),
    "reference_read_correspondences_s": t_ref, "reference_MB_s": mb / t_ref,
    "device_file_s": t_file, "device_file_MB_s": mb / t_file,
    "device_from_pinned_s": t_mem, "device_from_pinned_MB_s": mb / t_mem,
    "device_stage_ms": k_ms,
    "speedup_file_vs_reference": t_ref / t_file,
}))
path.unlink()

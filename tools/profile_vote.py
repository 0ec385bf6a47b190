"""Runs a few C3 device solves (for ncu captures of the vote kernel)."""
import sys
from pathlib import Path
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import torch  # noqa: E402
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

key = sys.argv[1] if len(sys.argv) > 1 else "c3"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
corrs, rots, _ = synth.make_config(key)
ctx = rv.Context(0)
d = torch.from_numpy(corrs).cuda()
for _ in range(reps):
    e = ctx.estimate_single_device(d.data_ptr(), corrs.shape[0], rv.EstimatorConfig())
torch.cuda.synchronize()
print("ok", e.inliers.size)

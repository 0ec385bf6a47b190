"""Dev probe: which adversarial constraints fail the vote's exactness guard (RV_STRICT_GUARD=1)."""
import os
import sys
from pathlib import Path

os.environ["RV_STRICT_GUARD"] = "1"
import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_2502_06337_b200 as rv  # noqa: E402

special = [[0, 0, 1], [0, 0, -1], [1, 0, 0], [0, 1, 0], [-1, 0, 0], [0, -1, 0],
           [1, 1, 0], [1, 0, 1], [0, 1, 1], [1e-7, 0, 1], [1e-4, 1e-4, 1], [0.6, 0.8, 0],
           [1, 1, 1], [-1, 1, 1e-12], [3e-4, 0, 1]]
z = np.array(special, dtype=np.float64)
z /= np.linalg.norm(z, axis=1, keepdims=True)
ctx = rv.Context(0)
for grid, samples in ((512, 2048), (256, 1024), (128, 512)):
    for i in range(len(z)):
        for rep in (1, 2):
            zz = np.repeat(z[i:i + 1], rep, axis=0)
            try:
                g = ctx.accumulate(zz, grid, 1.05, samples)
                ok = int(g.sum()) == rep * samples
                if not ok:
                    print(grid, samples, i, special[i], rep, "SUM", int(g.sum()))
            except Exception as e:  # noqa: BLE001
                print(grid, samples, i, special[i], rep, "ERR", str(e)[:200])
    zall = np.concatenate([z, z[:5]])
    try:
        ctx.accumulate(zall, grid, 1.05, samples)
        print(grid, samples, "all: ok")
    except Exception as e:  # noqa: BLE001
        print(grid, samples, "all: ERR", str(e)[:200])

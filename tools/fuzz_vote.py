"""Dev fuzzer: device accumulate vs the oracle (bit-exact) under RV_STRICT_GUARD=1 over random
geometries (grid, extent, samples) and adversarial constraint families: uniform, near-polar,
near-equatorial, near-axis-aligned, tiny perturbations of special directions, circles tangent to
random row boundaries. Prints every mismatch / guard failure; exit code 1 if any."""
import os
import sys
import time
from pathlib import Path

os.environ["RV_STRICT_GUARD"] = "1"
import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402
import paper_2502_06337_b200 as rv  # noqa: E402

rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 7)
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 240.0
ctx = rv.Context(0)
port = orc.Oracle("port")


def unit(v):
    return v / np.linalg.norm(v, axis=1, keepdims=True)


def family(kind, n, grid, extent):
    if kind == "uniform":
        return unit(rng.normal(size=(n, 3)))
    if kind == "polar":  # z near +-e3
        v = np.zeros((n, 3))
        v[:, 2] = rng.choice([-1.0, 1.0], n)
        v[:, :2] = rng.normal(size=(n, 2)) * 10.0 ** rng.uniform(-9, -2, (n, 1))
        return unit(v)
    if kind == "equatorial":  # z near the xy plane
        v = rng.normal(size=(n, 3))
        v[:, 2] *= 10.0 ** rng.uniform(-12, -2, n)
        return unit(v)
    if kind == "axis":  # near +-e1, +-e2, +-e3 and diagonals
        base = np.array([[1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0], [1, 0, 1], [0, 1, 1], [1, 1, 1]], float)
        v = base[rng.integers(0, len(base), n)] * rng.choice([-1.0, 1.0], (n, 3))
        v += rng.normal(size=(n, 3)) * 10.0 ** rng.uniform(-15, -3, (n, 1))
        return unit(v)
    if kind == "tangent":  # image circles tangent to random row boundaries
        cs = 2.0 * extent / grid
        out = []
        while len(out) < n:
            r = rng.integers(1, grid)
            y0 = -extent + r * cs
            if abs(y0) >= 0.999 or abs(y0) < 1e-9:
                continue
            cx = rng.uniform(-0.9, 0.9) * np.sqrt(1 - y0 * y0)
            top = rng.random() < 0.5
            cy = (y0 * y0 - 1 - cx * cx) / (2 * y0) if top else (1 + cx * cx - y0 * y0) / (2 * y0)
            rad = np.sqrt(1 + cx * cx + cy * cy)
            if (top and y0 - cy <= 0) or (not top and cy - y0 <= 0):
                continue
            nz = 1.0 / rad
            out.append([-cx * nz, -cy * nz, nz])
        return unit(np.array(out))
    raise ValueError(kind)


geoms = [(512, 1.05, 2048), (256, 1.05, 1024), (128, 1.05, 512), (200, 0.9, 1024), (1024, 1.05, 4096),
         (384, 1.2, 1536), (640, 1.0, 2048), (97, 1.3, 640), (512, 0.5, 1024), (300, 1.05, 768)]
kinds = ["uniform", "polar", "equatorial", "axis", "tangent"]
t0 = time.time()
fails = 0
trials = 0
while time.time() - t0 < budget:
    g = geoms[rng.integers(len(geoms))]
    k = kinds[rng.integers(len(kinds))]
    n = int(rng.integers(1, 3000))
    z = family(k, n, g[0], g[1])
    try:
        dev = ctx.accumulate(z, *g)
        ref = port.accumulate(z, *g)
        if not np.array_equal(dev, ref):
            fails += 1
            d = np.argwhere(dev != ref)
            print(f"MISMATCH geom={g} kind={k} n={n} cells={len(d)} first={d[:3].tolist()}", flush=True)
            np.save(f"gpurun_out/fuzz_fail_{fails}.npy", z)
    except Exception as e:  # noqa: BLE001
        fails += 1
        print(f"ERROR geom={g} kind={k} n={n}: {str(e)[:160]}", flush=True)
        np.save(f"gpurun_out/fuzz_fail_{fails}.npy", z)
    trials += 1
print(f"trials={trials} fails={fails} in {time.time() - t0:.0f}s")
sys.exit(1 if fails else 0)

"""Dev fuzzer: full estimates on the device (estimate_single device + host input, estimate_multi)
vs the oracle on random scenes (size, outlier fraction, noise, models, config) under
RV_STRICT_GUARD=1: identical inlier sets and axis votes, rotations within 1e-3 degrees, the same
error class when the reference throws. Prints every difference; exit code 1 if any."""
import os
import sys
import time
from pathlib import Path

os.environ["RV_STRICT_GUARD"] = "1"
import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402
import paper_2502_06337_b200 as rv  # noqa: E402
from paper_2502_06337_b200 import synth  # noqa: E402

seed = int(sys.argv[1]) if len(sys.argv) > 1 else 3
budget = float(sys.argv[2]) if len(sys.argv) > 2 else 240.0
rng = np.random.default_rng(seed)
ctx = rv.Context(0)
port = orc.Oracle("port")
t0 = time.time()
fails = trials = 0


def cmp(tag, dev, ref):
    global fails
    if not np.array_equal(dev.inliers, ref["inliers"]) or dev.axis_votes != ref["axis_votes"] or \
            orc.rotation_error_deg(dev.rotation, ref["rotation"]) > 1e-3:
        fails += 1
        print(f"DIFF {tag}: inl {dev.inliers.size}/{ref['inliers'].size} votes {dev.axis_votes}/{ref['axis_votes']} "
              f"rot {orc.rotation_error_deg(dev.rotation, ref['rotation']):.2e}", flush=True)
        return False
    return True


while time.time() - t0 < budget:
    n = int(10 ** rng.uniform(2, 5.3))
    models = int(rng.choice([1, 1, 1, 2, 3]))
    outl = float(rng.uniform(0.3, 0.97))
    sigma = float(10 ** rng.uniform(-4, -1.3))
    sc = int(rng.integers(1 << 30))
    if models == 1:
        corrs, _, _ = synth.make_scene(n, outl, sigma, seed=sc)
    else:
        corrs, _, _ = synth.make_scene(n, outl, sigma, models=models, model_frac=(1 - outl) / models, seed=sc)
    if rng.random() < 0.1:  # some degenerate pairs (x ~ y)
        k = rng.integers(0, n, max(1, n // 20))
        corrs[k, 3:] = corrs[k, :3] * (1 + 1e-12)
    cfg = rv.EstimatorConfig()
    ocfg = orc.default_config()
    if rng.random() < 0.3:
        cfg.grid = ocfg.grid = int(rng.choice([128, 256, 384, 512, 1024]))
        cfg.theta_samples = ocfg.theta_samples = int(rng.choice([512, 1024, 2048]))
    if rng.random() < 0.2:
        cfg.epsilon = ocfg.epsilon = float(rng.uniform(0.005, 0.05))
    tag = f"n={n} models={models} outl={outl:.2f} sigma={sigma:.1e} seed={sc} G={cfg.grid} J={cfg.theta_samples} eps={cfg.epsilon:.3f}"
    trials += 1
    try:
        ref = port.estimate_single(corrs, ocfg)
    except Exception as e:  # noqa: BLE001
        ref = e
    for mode in ("host", "device"):
        try:
            if mode == "host":
                dev = ctx.estimate_single(corrs, cfg)
            else:
                d = torch.from_numpy(corrs).cuda()
                dev = ctx.estimate_single_device(d.data_ptr(), n, cfg)
        except Exception as e:  # noqa: BLE001
            dev = e
        if isinstance(ref, Exception) or isinstance(dev, Exception):
            if type(ref).__name__ != type(dev).__name__ and not (isinstance(ref, Exception) and isinstance(dev, Exception)):
                fails += 1
                print(f"EXC {mode} {tag}: ref={type(ref).__name__}:{str(ref)[:80]} dev={type(dev).__name__}:{str(dev)[:80]}", flush=True)
            continue
        cmp(f"single/{mode} {tag}", dev, ref)
    if models > 1:
        mcfg = rv.EstimatorConfig(max_models=models + 1)
        mocfg = orc.default_config(max_models=models + 1)
        try:
            mref = port.estimate_multi(corrs, mocfg)
        except Exception as e:  # noqa: BLE001
            mref = e
        try:
            mdev = ctx.estimate_multi(corrs, mcfg)
        except Exception as e:  # noqa: BLE001
            mdev = e
        if isinstance(mref, Exception) or isinstance(mdev, Exception):
            rn = str(mref).split(":")[-1].strip() if isinstance(mref, Exception) else "ok"
            dn = type(mdev).__name__ if isinstance(mdev, Exception) else "ok"
            if not (isinstance(mref, Exception) and isinstance(mdev, Exception) and rn.lower() in dn.lower() + str(mdev).lower()):
                fails += 1
                print(f"MULTI EXC ref={str(mref)[:60]} dev={dn}:{str(mdev)[:60]} {tag}", flush=True)
        elif len(mref) != len(mdev):
            fails += 1
            print(f"MULTI count {len(mdev)}/{len(mref)} {tag}", flush=True)
        else:
            for k, (a, b) in enumerate(zip(mdev, mref)):
                cmp(f"multi[{k}] {tag}", a, b)
print(f"trials={trials} fails={fails} in {time.time() - t0:.0f}s")
sys.exit(1 if fails else 0)

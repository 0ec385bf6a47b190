"""Generates tests/golden/*.npz from the REFERENCE ITSELF (oracle/_ref: the unmodified
/root/reference sources compiled with the Eigen-subset shim, parity flags). Run in the build
container (needs /root/reference); the fixtures are committed and travel to the GPU box.

  fixture300.npz  the reference's bundled known-answer scene (proj/data/fixture_300.csv) and
                  the reference estimate on it (acceptance C8, test_output.txt:13: 0.271442 deg)
  cN.npz          BASELINE configs (paper_2502_06337_b200.synth, seeded) at parity sizes:
                  vote grid (or its sha256), top-3 NMS peaks, blurred argmax, estimate(s)
"""
from __future__ import annotations

import hashlib
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "oracle"))
import oracle as orc  # noqa: E402

from paper_2502_06337_b200 import synth  # noqa: E402

OUT = Path(__file__).resolve().parent
REF_FIXTURE = Path("/root/reference/proj/data")

SIZES = {"c1": 1000, "c2": 20000, "c3": 20000, "c4": 20000, "c5": 20000}


def est_arrays(prefix: str, e: dict) -> dict:
    return {f"{prefix}axis": e["axis"], f"{prefix}angle": np.float64(e["angle"]), f"{prefix}rotation": e["rotation"],
            f"{prefix}axis_votes": np.uint32(e["axis_votes"]), f"{prefix}inliers": e["inliers"].astype(np.int32)}


def read_fixture_csv(path: Path) -> np.ndarray:
    rows = []
    for k, line in enumerate(path.read_text().splitlines()):
        if k == 0 and not line[:1].lstrip("-").replace(".", "").isdigit():
            continue
        if line.strip():
            rows.append([float(v) for v in line.split(",")])
    return np.array(rows, dtype=np.float64)


def main() -> None:
    ref = orc.Oracle("ref_parity")
    # bundled fixture
    corrs = read_fixture_csv(REF_FIXTURE / "fixture_300.csv")
    truth_lines = (REF_FIXTURE / "fixture_300_truth.txt").read_text().split("\n")
    r_truth = np.array([float(v) for v in truth_lines[1].split()]).reshape(3, 3)
    labels = np.array([int(v) for v in truth_lines[3].split()])
    e = ref.estimate_single(corrs)
    np.savez_compressed(OUT / "fixture300.npz", corrs=corrs, r_truth=r_truth, labels=labels,
                        ref_err_deg=np.float64(0.271442), **est_arrays("est_", e))
    print("fixture300: err vs truth", orc.rotation_error_deg(r_truth, e["rotation"]), "inliers", e["inliers"].size)
    for key, n in SIZES.items():
        corrs, rots, labels = synth.make_config(key, n)
        z, kept, dropped = ref.preprocess(corrs)
        grid = ref.accumulate(z)
        peaks = ref.find_peaks(grid, 3, 8, 1)
        blur = [ref.blurred_argmax(grid, r) for r in (4, 8, 16, 32, 64)]
        arrays = {"n": np.int64(n), "z_sha256": np.frombuffer(hashlib.sha256(z.tobytes()).digest(), np.uint8),
                  "n_kept": np.int64(z.shape[0]),
                  "grid_sha256": np.frombuffer(hashlib.sha256(grid.tobytes()).digest(), np.uint8),
                  "grid_total": np.uint64(grid.sum(dtype=np.uint64)),
                  "peaks": np.array([[p[0], p[1], p[4]] for p in peaks], np.int64),
                  "blur": np.array([[b[0], b[1], b[4]] for b in blur], np.int64)}
        if key == "c1":
            arrays["grid"] = grid
        if key == "c5":
            cfg = orc.default_config(max_models=3)
            ms = ref.estimate_multi(corrs, cfg)
            arrays["n_models"] = np.int64(len(ms))
            for k, m in enumerate(ms):
                arrays.update(est_arrays(f"m{k}_", m))
        else:
            arrays.update(est_arrays("est_", ref.estimate_single(corrs)))
        np.savez_compressed(OUT / f"{key}.npz", **arrays)
        print(key, "n", n, "grid total", int(arrays["grid_total"]), "peaks", arrays["peaks"].tolist())


if __name__ == "__main__":
    main()

"""Seeded synthetic correspondences for the five BASELINE.json configurations.

BASELINE.json names no public dataset; these generators follow its stated shapes and
distributions: p_i ~ N(0, I3); R from a normalised Gaussian
quaternion; inliers q_i = R p_i + N(0, sigma^2 I3); outliers q_i ~ N(0, I3) at seeded random
positions; multi-rotation: K rotations at pairwise geodesic distance >= 30 degrees.
numpy's PCG64 makes the draw reproducible across machines. Rows are (x0 x1 x2 y0 y1 y2),
float64, C-contiguous -- the reference's span<const Correspondence> layout.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

BASE_SEED = 250206337


@dataclass(frozen=True)
class SceneConfig:
    name: str
    n: int
    outlier_frac: float
    sigma: float
    models: int = 1
    model_frac: float = 0.0   # inlier fraction per model (multi-rotation); 0 = 1 - outlier_frac
    seed: int = BASE_SEED
    max_models: int = 1       # estimator max_models for this config


CONFIGS = {
    "c1": SceneConfig("c1_n1e3_out50_s0.01", 1_000, 0.50, 0.01, seed=BASE_SEED + 1),
    "c2": SceneConfig("c2_n1e5_out90_s0.01", 100_000, 0.90, 0.01, seed=BASE_SEED + 2),
    "c3": SceneConfig("c3_n1e6_out90_s0.01", 1_000_000, 0.90, 0.01, seed=BASE_SEED + 3),
    "c4": SceneConfig("c4_n1e6_out99_s0.05", 1_000_000, 0.99, 0.05, seed=BASE_SEED + 4),
    "c5": SceneConfig("c5_n1e6_k3_out85_s0.01", 1_000_000, 0.85, 0.01, models=3, model_frac=0.05,
                      seed=BASE_SEED + 5, max_models=3),
}


def quat_to_rot(q: np.ndarray) -> np.ndarray:
    w, x, y, z = q / np.linalg.norm(q)
    return np.array([
        [1 - 2 * (y * y + z * z), 2 * (x * y - z * w), 2 * (x * z + y * w)],
        [2 * (x * y + z * w), 1 - 2 * (x * x + z * z), 2 * (y * z - x * w)],
        [2 * (x * z - y * w), 2 * (y * z + x * w), 1 - 2 * (x * x + y * y)],
    ])


def geodesic(r1: np.ndarray, r2: np.ndarray) -> float:
    c = 0.5 * (np.trace(r1.T @ r2) - 1.0)
    return float(np.arccos(np.clip(c, -1.0, 1.0)))


def make_scene(n: int, outlier_frac: float, sigma: float, models: int = 1, model_frac: float = 0.0,
               seed: int = BASE_SEED, min_sep_deg: float = 30.0):
    """Returns (corrs (n, 6) float64, rotations list of (3, 3), labels (n,) int: model id or -1)."""
    rng = np.random.default_rng(seed)
    rots: list[np.ndarray] = []
    while len(rots) < models:
        r = quat_to_rot(rng.normal(size=4))
        if all(geodesic(r, q) >= np.deg2rad(min_sep_deg) for q in rots):
            rots.append(r)
    if models == 1 and model_frac == 0.0:
        counts = [n - int(round(outlier_frac * n))]
    else:
        counts = [int(round(model_frac * n))] * models
    labels = np.full(n, -1, np.int64)
    pos = 0
    for k, cnt in enumerate(counts):
        labels[pos:pos + cnt] = k
        pos += cnt
    labels = labels[rng.permutation(n)]
    p = rng.normal(size=(n, 3))
    q_out = rng.normal(size=(n, 3))
    noise = rng.normal(size=(n, 3)) * sigma
    y = q_out.copy()
    for k, r in enumerate(rots):
        m = labels == k
        y[m] = p[m] @ r.T + noise[m]
    corrs = np.ascontiguousarray(np.concatenate([p, y], axis=1))
    return corrs, rots, labels


def make_config(key: str, n: int | None = None):
    """Scene of BASELINE config `key` ("c1".."c5"); `n` overrides the size (same generator)."""
    c = CONFIGS[key]
    return make_scene(n or c.n, c.outlier_frac, c.sigma, c.models, c.model_frac, c.seed)

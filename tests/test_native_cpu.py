"""CPU: the C-ABI library loads, exports every entry point declared in include/*.h, its host
arithmetic (geometry, vote floor) equals the reference formulas, and without a GPU it fails
loudly (no CPU fallback)."""
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

import paper_2502_06337_b200 as rv
from paper_2502_06337_b200 import _native

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols() -> set:
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        names |= set(re.findall(r"\b(rv_[a-z0-9_]+)\s*\(", h.read_text()))
    return names


def test_library_exports_every_declared_symbol():
    lib = _native.LIB_PATH
    assert lib.exists(), "build the library first (__graft_entry__.build())"
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib)], capture_output=True, text=True, check=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if " T " in ln}
    missing = declared_symbols() - exported
    assert not missing, f"declared but not exported: {sorted(missing)}"
    assert declared_symbols() == set(_native.EXPORTED_SYMBOLS)


def test_library_is_sm100a():
    out = subprocess.run(["cuobjdump", "-lelf", str(_native.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_abi_and_defaults():
    lib = _native.lib()
    assert lib.rv_abi_version() == 5
    c = _native.rv_config()
    lib.rv_config_default(c)
    d = rv.EstimatorConfig()
    for f, _ in _native.rv_config._fields_:
        assert getattr(c, f) == (int(getattr(d, f)) if isinstance(getattr(d, f), bool) else getattr(d, f)), f


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(rv.errors.DeviceError):
        rv.Context(0)


def test_geometry_fixtures():
    # geom.cpp / test_geom.cpp fixtures
    assert np.allclose(rv.rodrigues([0, 0, 1], np.pi / 2) @ [1, 0, 0], [0, 1, 0], atol=1e-12)
    half = rv.rodrigues([0, 0, 1], np.pi)
    assert np.allclose(half, np.diag([-1, -1, 1]), atol=1e-12)
    assert rv.rotation_error(np.eye(3), half) == pytest.approx(np.pi)
    assert rv.project([0, 0.6, -0.8]) == pytest.approx((0.0, 1.0 / 3.0))
    with pytest.raises(rv.PoleProximity):
        rv.project([0, 0, 1])
    assert np.allclose(rv.unproject(1.0, 0.0), [1, 0, 0], atol=1e-12)
    assert np.array_equal(rv.canonicalize([0, 0.6, 0.8]), [0, -0.6, -0.8])
    a1, a2 = rv.orthonormal_basis([0, 0, 1])
    assert abs(a1 @ a2) < 1e-12 and abs(a1[2]) < 1e-12 and abs(a2[2]) < 1e-12
    assert rv.correspondence_angle([0, 0, 1], [1, 0, 0], [0, 1, 0]) == pytest.approx(np.pi / 2, rel=1e-12)
    with pytest.raises(rv.DegenerateProjection):
        rv.correspondence_angle([0, 0, 1], [0, 0, 1], [1, 0, 0])


def test_rodrigues_matches_oracle_bitwise():
    import ctypes as C
    import oracle as orc
    port = orc.Oracle("port")
    rng = np.random.default_rng(3)
    for _ in range(100):
        ax = rng.normal(size=3)
        ax /= np.linalg.norm(ax)
        ang = rng.uniform(-np.pi, np.pi)
        r = np.empty(9)
        port.lib.rvo_rodrigues(ax.ctypes.data_as(C.POINTER(C.c_double)), C.c_double(ang),
                               r.ctypes.data_as(C.POINTER(C.c_double)))
        assert np.array_equal(rv.rodrigues(ax, ang).reshape(9), r)


def test_peak_vote_floor_formula():
    cfg = rv.EstimatorConfig()
    # estimator.cpp:311-318 at N=1e6: 0.02 * 1e6 * 2048 * (2.1/512) / (2 pi)
    assert rv.peak_vote_floor(cfg, 1_000_000) == int(0.02 * 1e6 * 2048 * (2 * 1.05 / 512) / (2 * np.pi))
    assert rv.peak_vote_floor(cfg, 10) == 16

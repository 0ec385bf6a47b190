"""Shared fixtures. `-m "not gpu"` runs here (no GPU); `-m gpu` runs on a B200 through the C-ABI."""
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
for p in (str(ROOT), str(ROOT / "oracle")):
    if p not in sys.path:
        sys.path.insert(0, p)


# a failed vote exactness guard (band-plan coverage bug) is an error in the tests, not a silent
# exact re-vote (rv_api.cpp guard_failed)
os.environ.setdefault("RV_STRICT_GUARD", "1")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a library")


@pytest.fixture(scope="session")
def port():
    import oracle as orc
    return orc.Oracle("port")


@pytest.fixture(scope="session")
def ref():
    import oracle as orc
    try:
        return orc.Oracle("ref_parity")
    except (FileNotFoundError, OSError) as e:
        pytest.skip(f"reference build unavailable: {e}")


@pytest.fixture(scope="session")
def ctx():
    import paper_2502_06337_b200 as rv
    return rv.Context(0)


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as f:
        return {k: f[k] for k in f.files}

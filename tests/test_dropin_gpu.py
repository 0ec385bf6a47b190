"""GPU: the reference's own unit suites (proj/tests/test_*.cpp, unmodified) and its callers of
the path (baselines.cpp, synth.cpp, io.cpp, bench.cpp) compiled against this repo's drop-in C++
headers and linked with librotavote_b200.so (tests/dropin/Makefile). Every call into
estimate_single / estimate_multi / accumulate / find_peaks / classify / refine / vote_angles in
those tests runs on the B200 kernels."""
import re
import subprocess
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
BIN = Path(__file__).resolve().parent / "_bin" / "ref_tests_on_b200"


def test_reference_unit_suites_on_b200():
    if not BIN.exists():
        pytest.skip("drop-in binary not built (needs /root/reference at build time)")
    res = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    out = res.stdout + res.stderr
    m = re.search(r"test cases: (\d+) \| (\d+) passed \| (\d+) failed \| assertions: (\d+) \| (\d+) failed", out)
    assert m, out[-2000:]
    cases, passed, failed, asserts, afailed = map(int, m.groups())
    print(out[-3000:])
    assert failed == 0 and afailed == 0 and cases >= 50, out[-3000:]

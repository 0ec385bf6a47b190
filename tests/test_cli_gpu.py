"""GPU: the reference's command-line tool (proj/tools/rotavote_cli.cpp, unmodified) built against
this repo's drop-in headers -- estimate / multi / dump-acc / oracle / bench run on the B200 library,
read_correspondences parses on the device, write_result / truth / dumps are include/rotavote/io.hpp
(tests/dropin/Makefile). The steps and checks restate the reference's end-to-end CLI test
(proj/tests/cli_roundtrip.cmake): synth -> estimate -> result document -> multi -> oracle ->
dump-acc PGM -> bench CSV shape -> a malformed CSV fails cleanly. Also checks the result document
round-trips bit-exact against the estimate printed by the C-ABI."""
import json
import re
import subprocess
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
CLI = Path(__file__).resolve().parent / "_bin" / "rotavote_cli_on_b200"


def run(*args, ok=True):
    r = subprocess.run([str(CLI), *map(str, args)], capture_output=True, text=True, timeout=300)
    if ok:
        assert r.returncode == 0, f"{args}: rc={r.returncode}\n{r.stdout}\n{r.stderr}"
    return r


@pytest.fixture(scope="module")
def work(tmp_path_factory):
    if not CLI.exists():
        pytest.skip("CLI not built (tests/dropin: make; needs /root/reference at build time)")
    return tmp_path_factory.mktemp("cli")


def test_cli_roundtrip(work, ctx):
    scene, truth = work / "scene.csv", work / "truth.txt"
    run("synth", "--n", 2000, "--rho", 0.4, "--sigma", 0.01, "--seed", 9001, "-o", scene, "--truth", truth)
    assert scene.exists() and truth.exists()
    assert truth.read_text().startswith("rotations 1\n")

    result = work / "result.json"
    out = run("estimate", "-i", scene, "-o", result).stdout
    assert "model 0: axis" in out
    doc = json.loads(result.read_text())
    assert len(doc) == 1 and "angle_rad" in doc[0]
    # the document holds exactly what the library computes for the same rows (bit-exact numbers)
    rows = np.loadtxt(scene, delimiter=",", skiprows=1)
    e = ctx.estimate_single(rows)
    assert doc[0]["inlier_indices"] == e.inliers.tolist() and doc[0]["inlier_count"] == e.inliers.size
    assert doc[0]["axis_votes"] == e.axis_votes
    assert np.array_equal(np.array(doc[0]["matrix"]), e.rotation.reshape(-1))
    assert doc[0]["angle_rad"] == e.angle

    out = run("multi", "-i", scene, "--max-models", 3).stdout
    assert "model 0: axis" in out

    out = run("oracle", "-i", scene, "--directions", 2000).stdout
    assert re.search(r"consensus [0-9]+", out)

    pgm = work / "acc.pgm"
    run("dump-acc", "-i", scene, "-o", pgm, "--format", "pgm", "--grid", 128)
    raw = pgm.read_bytes()
    assert raw.startswith(b"P5\n128 128\n255\n") and len(raw) == len(b"P5\n128 128\n255\n") + 128 * 128

    bench = work / "bench.csv"
    run("bench", "--n", 500, "--rho", 0.3, "--trials", 2, "--estimators", "vote", "ransac",
        "--grid", 256, "--theta-samples", 1024, "-o", bench)
    lines = bench.read_text().splitlines()
    assert lines[0] == "scenario,trial,estimator,n,rho,sigma,e_rot_deg,time_s,success"
    assert len(lines) == 7  # header + 2x2 trials + 2 aggregate rows

    bad = work / "bad.csv"
    bad.write_text("1,0,0,0,1\n")
    r = run("estimate", "-i", bad, ok=False)
    assert r.returncode != 0 and "error:" in r.stderr


def test_cli_text_dump_conserves_votes(work):
    scene = work / "s2.csv"
    run("synth", "--n", 300, "--rho", 0.5, "--sigma", 0.01, "--seed", 5, "-o", scene)
    txt = work / "acc.txt"
    run("dump-acc", "-i", scene, "-o", txt, "--format", "text", "--grid", 64, "--theta-samples", 256)
    g = np.loadtxt(txt, dtype=np.uint64)
    assert g.shape == (64, 64) and int(g.sum()) == 300 * 256  # no degenerate pairs at rho 0.5

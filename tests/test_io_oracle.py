"""CPU: the CSV oracle (the reference's own read_correspondences, io.cpp:66-101, compiled into
oracle/_ref) on the reference's io fixtures (test_io_bench.cpp:45-88)."""
import numpy as np
import pytest


def test_reference_csv_fixtures(ref, tmp_path):
    p = tmp_path / "a.csv"
    p.write_text("1,0,0,0,1,0\n0,1,0,-1,0,0\n")
    rows, err = ref.read_correspondences(p)
    assert err is None and np.array_equal(rows, [[1, 0, 0, 0, 1, 0], [0, 1, 0, -1, 0, 0]])
    p.write_text("x0,x1,x2,y0,y1,y2\n1,0,0,0,1,0\n")
    rows, err = ref.read_correspondences(p)
    assert err is None and rows.shape == (1, 6)
    p.write_text("1,0,0,0,1,0\n1,0,0,0,1\n")
    rows, err = ref.read_correspondences(p)
    assert rows is None and err == ("ParseError", "expected 6 fields, got 5 (line 2)", 2)
    p.write_text("")
    assert ref.read_correspondences(p)[1][0] == "EmptyFile"
    assert ref.read_correspondences(tmp_path / "missing.csv")[1][0] == "IoError"

"""CSV ingest on the device vs the reference's own
read_correspondences (io.cpp:66-101, compiled from /root/reference into oracle/_ref): identical
rows bit for bit, identical error kind / message / line. Fixtures mirror the reference's
test_io_bench.cpp:45-88; the stress sets cover the exact decimal->binary fast path and every
host-fallback class (more than 19 digits, subnormals, overflow, inf/nan)."""
import numpy as np
import pytest

import paper_2502_06337_b200 as rv
from paper_2502_06337_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ctx():
    return rv.Context(0)


def run_both(ctx, ref, path):
    """(device rows | device error, reference rows | reference error)."""
    try:
        dev = ("ok", ctx.read_correspondences(path))
    except rv.ParseError as e:
        dev = ("ParseError", str(e), e.line)
    except rv.EmptyFile as e:
        dev = ("EmptyFile", str(e).split(": ", 1)[-1], 0)
    except rv.IoError as e:
        dev = ("IoError", str(e).split(": ", 1)[-1], 0)
    rows, err = ref.read_correspondences(path)
    refr = ("ok", rows) if err is None else err
    return dev, refr


def assert_same(dev, refr):
    assert dev[0] == refr[0], (dev, refr)
    if dev[0] == "ok":
        assert dev[1].shape == refr[1].shape
        assert np.array_equal(dev[1].view(np.uint64), refr[1].view(np.uint64))  # bit-exact (incl. -0.0)
    elif dev[0] == "ParseError":
        assert dev[1] == refr[1] and dev[2] == refr[2]
    else:
        assert dev[1] == refr[1]


def write(tmp_path, name, text):
    p = tmp_path / name
    p.write_bytes(text.encode() if isinstance(text, str) else text)
    return p


@pytest.mark.parametrize("text", [
    "1,0,0,0,1,0\n0,1,0,-1,0,0\n",                      # plain rows
    "x0,x1,x2,y0,y1,y2\n1,0,0,0,1,0\n",                 # header skipped
    "1,0,0,0,1,0\n1,0,0,0,1\n",                         # short row -> line 2
    "1,0,0,0,1,0\n1,zero,0,0,1,0\n",                    # not a number -> line 2
    "",                                                 # EmptyFile (no data)
    "x0,x1,x2,y0,y1,y2\n",                              # EmptyFile (no rows)
    "\n  \n\t\n",                                       # blank lines only
    "1,2,3,4,5,6",                                      # no final newline
    "1,2,3,4,5,6\r\n\r\n7,8,9,10,11,12\r\n",            # CRLF + blank CRLF line
    " 1 ,\t2,3 ,4,5,6\n",                               # field whitespace
    "1,2,3,4,5,6\n,2,3,4,5,6\n",                        # empty field
    "1,2,3,4,5,6\n1,2,3,4,5,6,7\n",                     # long row
    "+1,2,3,4,5,6\n",                                   # leading '+': from_chars rejects
    "1e,2,3,4,5,6\n",                                   # dangling exponent
    "0x10,2,3,4,5,6\n",                                 # hex is not general format
    ".5,5.,-.5,-0,0.0e0,1E+2\n",                        # forms from_chars accepts
    "1,2,3,4,5,6\n\n\nx,2,3,4,5,6\n",                   # header test only on line 1
    "x0,x1\n1,2,3,4,5,6\n",                             # header with any field count
    "  \nx0,x1,x2,y0,y1,y2\n1,2,3,4,5,6\n",             # blank line 1: line 2 is not a header
    "1,2,3,4,5,6\r\r\n",                                # only one '\r' is stripped
    "inf,-inf,nan,Infinity,1,2\n",                      # from_chars specials (host fallback)
    "1e400,2,3,4,5,6\n",                                # overflow (host fallback decides)
    "4.9406564584124654e-324,2.2250738585072014e-308,1.7976931348623157e308,1e-320,0,0\n",
    "12345678901234567890123,0.1234567890123456789012,1,2,3,4\n",  # > 19 digits
    "9007199254740993,9007199254740995,1e23,8.533e-309,2.5e-324,3e-324\n",  # rounding edges
])
def test_fixture_parity(ctx, ref, tmp_path, text):
    assert_same(*run_both(ctx, ref, write(tmp_path, "f.csv", text)))


def test_missing_file(ctx, ref, tmp_path):
    assert_same(*run_both(ctx, ref, tmp_path / "missing.csv"))


def test_round_trip_of_the_reference_writer_format(ctx, ref, tmp_path):
    # write_correspondences (io.cpp:103-110): header + %.17g; a C3-sized sample
    corrs, _, _ = synth.make_config("c3", 300_000)
    lines = ["x0,x1,x2,y0,y1,y2"] + [",".join("%.17g" % v for v in row) for row in corrs]
    p = write(tmp_path, "c3.csv", "\n".join(lines) + "\n")
    dev, refr = run_both(ctx, ref, p)
    assert_same(dev, refr)
    assert np.array_equal(dev[1].view(np.uint64), corrs.view(np.uint64))  # bit-exact round trip


def random_literals(rng, n):
    """Decimal literals over the whole binary64 range in the forms a CSV writer produces."""
    out = []
    bits = rng.integers(0, 2**63, size=n, dtype=np.int64).astype(np.uint64) | (
        rng.integers(0, 2, size=n).astype(np.uint64) << np.uint64(63))
    vals = bits.view(np.float64)
    vals = vals[np.isfinite(vals)]
    for k, v in enumerate(vals):
        m = k % 6
        if m == 0:
            out.append(repr(float(v)))                        # shortest round trip
        elif m == 1:
            out.append("%.17g" % v)
        elif m == 2:
            out.append("%.6e" % v)                            # rounded: exercises correct rounding
        elif m == 3:
            d = int(rng.integers(1, 20))                      # 1..19 significant digits, normal range
            out.append(f"{int(rng.integers(0, 10**d, dtype=np.uint64))}e{int(rng.integers(-300, 300 - d))}")
        elif m == 4:
            out.append("%.19e" % v)                           # 20 digits: host fallback
        else:
            out.append("%.3f" % (v * 1e-300) if abs(v) < 1e300 else "%.3g" % v)
    return out


def test_random_literals_bit_exact(ctx, ref, tmp_path):
    rng = np.random.default_rng(2024)
    lits = random_literals(rng, 240_000)
    lits = lits[: len(lits) // 6 * 6]
    rows = [",".join(lits[i:i + 6]) for i in range(0, len(lits), 6)]
    path = write(tmp_path, "r.csv", "\n".join(rows) + "\n")
    dev, refr = run_both(ctx, ref, path)
    assert dev[0] == "ok" and dev[1].shape[0] == len(rows)  # rows compared, not just an error
    assert_same(dev, refr)

def test_host_fallback_fields_are_counted(ctx):
    # fields outside the device's exact fast path (subnormal results, a decimal halfway between
    # two doubles) are parsed by the host's from_chars and counted
    ctx.parse_correspondences_device(b"4.9e-324,2.5e-320,9007199254740993,1,2,3\n3,4,5,6,7,8\n")
    assert ctx.stage_times()["csv_host_fields"] >= 2
    ctx.parse_correspondences_device(b"1,2,3,4,5,6\n")
    assert ctx.stage_times()["csv_host_fields"] == 0


def test_first_error_line_wins_across_paths(ctx, ref, tmp_path):
    # an error inside a host-fallback field (line 4) before a device syntax error (line 6)
    rows = ["1,2,3,4,5,6"] * 8
    rows[3] = "1e999999,2,3,4,5,6"       # out of range: from_chars error, found by the host
    rows[5] = "1,2,3,4,5,abc"            # syntax error, found by the device
    assert_same(*run_both(ctx, ref, write(tmp_path, "e.csv", "\n".join(rows) + "\n")))


def test_device_rows_feed_the_solver(ctx, tmp_path):
    corrs, _, _ = synth.make_config("c2", 20_000)
    lines = [",".join("%.17g" % v for v in row) for row in corrs]
    p = write(tmp_path, "s.csv", "\n".join(lines) + "\n")
    dptr, n = ctx.read_correspondences_device(str(p))
    assert n == corrs.shape[0]
    e_dev = ctx.estimate_single_device(dptr, n)
    e_host = ctx.estimate_single(corrs)
    assert np.array_equal(e_dev.inliers, e_host.inliers) and np.array_equal(e_dev.rotation, e_host.rotation)


def test_parse_from_memory_matches_file(ctx, ref, tmp_path):
    corrs, _, _ = synth.make_config("c1")
    text = ("x0,x1,x2,y0,y1,y2\r\n" + "\r\n".join(",".join(repr(float(v)) for v in r) for r in corrs)).encode()
    rows_mem = ctx.parse_correspondences(text)
    rows_file, err = ref.read_correspondences(write(tmp_path, "m.csv", text))
    assert err is None and np.array_equal(rows_mem.view(np.uint64), rows_file.view(np.uint64))
    assert np.array_equal(rows_mem.view(np.uint64), corrs.view(np.uint64))
    with pytest.raises(rv.ParseError) as e:
        ctx.parse_correspondences(b"1,2,3,4,5,6\n1,2,3\n")
    assert e.value.line == 2 and "expected 6 fields, got 3" in str(e.value)

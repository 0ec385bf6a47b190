"""ctypes access to the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Two checkers with one API:
  * ``Oracle("port")``: the plain-C restatement oracle/rv_oracle.c (liboracle.so);
  * ``Oracle("ref_parity")`` / ``Oracle("ref_perf")``: the UNMODIFIED reference sources compiled
    from /root/reference with the Eigen-subset shim (oracle/_ref/librotavote_ref_*.so), parity
    flavour (-O2 -ffp-contract=off) or the reference's own flags (-O3 -march=native).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm may use this
module, and only as the checker -- never as the measured or shipped path.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_LIB = HERE / "liboracle.so"
REF_LIBS = {"ref_parity": HERE / "_ref" / "librotavote_ref_parity.so",
            "ref_perf": HERE / "_ref" / "librotavote_ref_perf.so"}

STATUS_NAMES = {0: "ok", 1: "EmptyInput", 2: "NoPeak", 3: "DegenerateProjection", 4: "NoVotes",
                5: "AllDegenerate", 6: "RankDeficient", 7: "NoConsensus", 8: "InvalidConfig",
                9: "PoleProximity", 10: "OutOfMemory", 99: "Unknown"}


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: {STATUS_NAMES.get(status, status)}")
        self.status = status
        self.name = STATUS_NAMES.get(status, str(status))


class Config(C.Structure):  # rvo_config / ref_config / rv_config (same layout)
    _fields_ = [("grid", C.c_int32), ("extent", C.c_double), ("theta_samples", C.c_int32),
                ("epsilon", C.c_double), ("angle_bins", C.c_int32), ("max_models", C.c_int32),
                ("min_votes_frac", C.c_double), ("consensus_floor_mult", C.c_double),
                ("dedupe_overlap", C.c_double), ("tau_z", C.c_double), ("tau_deg", C.c_double),
                ("suppression_radius", C.c_int32), ("refine", C.c_int32), ("normalize_inputs", C.c_int32),
                ("threads", C.c_int32)]


class PeakS(C.Structure):
    _fields_ = [("ix", C.c_int32), ("iy", C.c_int32), ("A", C.c_double), ("B", C.c_double), ("votes", C.c_uint32)]


class EstPort(C.Structure):
    _fields_ = [("axis", C.c_double * 3), ("angle", C.c_double), ("rotation", C.c_double * 9),
                ("axis_votes", C.c_uint32), ("n_inliers", C.c_int64), ("inliers", C.POINTER(C.c_int32))]


class EstRef(C.Structure):
    _fields_ = EstPort._fields_ + [("elapsed_s", C.c_double)]


class Trace(C.Structure):
    _fields_ = [("peak_ix", C.c_int32), ("peak_iy", C.c_int32), ("peak_votes", C.c_uint32),
                ("start_axis", C.c_double * 3), ("refine_passes", C.c_int32), ("rescued", C.c_int32),
                ("rescue_won", C.c_int32), ("n_kept", C.c_int64), ("n_dropped", C.c_int64)]


def build_port(force: bool = False) -> Path:
    """Compiles the C restatement (gcc, strict IEEE order)."""
    src = HERE / "rv_oracle.c"
    if force or not PORT_LIB.exists() or PORT_LIB.stat().st_mtime < max(src.stat().st_mtime,
                                                                        (HERE / "rv_oracle.h").stat().st_mtime):
        subprocess.run(["gcc", "-O2", "-ffp-contract=off", "-std=c11", "-fPIC", "-shared", "-o", str(PORT_LIB),
                        str(src), "-lm"], check=True)
    return PORT_LIB


def default_config(**kw) -> Config:
    c = Config(512, 1.05, 2048, 0.015, 1024, 1, 0.02, 1.5, 0.5, 1e-9, 1e-6, 8, 1, 1, 1)
    for k, v in kw.items():
        setattr(c, k, int(v) if isinstance(v, bool) else v)
    return c


def _p(a, t):
    return a.ctypes.data_as(C.POINTER(t))


class Oracle:
    def __init__(self, kind: str = "port"):
        self.kind = kind
        if kind == "port":
            self.lib = C.CDLL(str(build_port()))
            self.pre = "rvo_"
        else:
            path = REF_LIBS[kind]
            if not path.exists():
                raise FileNotFoundError(f"{path} not built (oracle/ref_build: make)")
            self.lib = C.CDLL(str(path))
            self.pre = "ref_"

    def _fn(self, name):
        return getattr(self.lib, self.pre + name)

    def _ck(self, st, what):
        if st != 0:
            raise OracleError(st, what)

    # ---- path functions ----------------------------------------------------------------
    def preprocess(self, corrs, tau_z=1e-9, normalize=True):
        a = np.ascontiguousarray(corrs, dtype=np.float64).reshape(-1, 6)
        n = a.shape[0]
        z = np.empty((max(n, 1), 3))
        kept = np.empty(max(n, 1), np.int32)
        dropped = np.empty(max(n, 1), np.int32)
        nk, nd = C.c_int64(), C.c_int64()
        f = self._fn("preprocess")
        f.restype = C.c_int
        st = f(_p(a, C.c_double), C.c_int64(n), C.c_double(tau_z), C.c_int(int(normalize)), _p(z, C.c_double),
               _p(kept, C.c_int32), _p(dropped, C.c_int32), C.byref(nk), C.byref(nd))
        self._ck(st, "preprocess")
        return z[:nk.value].copy(), kept[:nk.value].copy(), dropped[:nd.value].copy()

    def accumulate(self, z, grid=512, extent=1.05, samples=2048, threads=1):
        zz = np.ascontiguousarray(z, dtype=np.float64).reshape(-1, 3)
        out = np.zeros((grid, grid), np.uint32)
        f = self._fn("accumulate")
        f.restype = C.c_int
        if self.kind == "port":
            st = f(_p(zz, C.c_double), C.c_int64(zz.shape[0]), C.c_int32(grid), C.c_double(extent),
                   C.c_int32(samples), _p(out, C.c_uint32))
        else:
            st = f(_p(zz, C.c_double), C.c_int64(zz.shape[0]), C.c_int32(grid), C.c_double(extent),
                   C.c_int32(samples), C.c_int32(threads), _p(out, C.c_uint32))
        self._ck(st, "accumulate")
        return out

    def find_peaks(self, counts, max_peaks, radius, min_votes, extent=1.05):
        g = np.ascontiguousarray(counts, dtype=np.uint32)
        out = (PeakS * max(1, max_peaks))()
        n = C.c_int32()
        f = self._fn("find_peaks")
        f.restype = C.c_int
        st = f(_p(g, C.c_uint32), C.c_int32(g.shape[0]), C.c_double(extent), C.c_int32(max_peaks),
               C.c_int32(radius), C.c_uint32(min_votes), out, C.byref(n))
        self._ck(st, "find_peaks")
        return [(out[k].ix, out[k].iy, out[k].A, out[k].B, out[k].votes) for k in range(n.value)]

    def blurred_argmax(self, counts, radius, extent=1.05):
        g = np.ascontiguousarray(counts, dtype=np.uint32)
        p = PeakS()
        f = self._fn("blurred_argmax")
        f.restype = C.c_int
        self._ck(f(_p(g, C.c_uint32), C.c_int32(g.shape[0]), C.c_double(extent), C.c_int32(radius), C.byref(p)),
                 "blurred_argmax")
        return (p.ix, p.iy, p.A, p.B, p.votes)

    def classify_inliers(self, axis, z, eps):
        ax = np.ascontiguousarray(axis, dtype=np.float64)
        zz = np.ascontiguousarray(z, dtype=np.float64).reshape(-1, 3)
        out = np.empty(max(zz.shape[0], 1), np.int32)
        f = self._fn("classify_inliers")
        f.restype = C.c_int64
        m = f(_p(ax, C.c_double), _p(zz, C.c_double), C.c_int64(zz.shape[0]), C.c_double(eps), _p(out, C.c_int32))
        return out[:m].copy()

    def refine_axis(self, z):
        zz = np.ascontiguousarray(z, dtype=np.float64).reshape(-1, 3)
        out = np.empty(3)
        f = self._fn("refine_axis")
        f.restype = C.c_int
        self._ck(f(_p(zz, C.c_double), C.c_int64(zz.shape[0]), _p(out, C.c_double)), "refine_axis")
        return out

    # ---- I/O (reference library only: io.cpp) ------------------------------------------------
    def read_correspondences(self, path):
        """The reference's read_correspondences (io.cpp:66-101): (rows, None) or (None, (kind,
        message, line)) with kind in {"ParseError", "EmptyFile", "IoError"}."""
        assert self.kind != "port", "I/O is checked against the compiled reference only"
        out = C.POINTER(C.c_double)()
        n, line = C.c_int64(), C.c_int64()
        msg = C.create_string_buffer(1024)
        f = self._fn("read_correspondences")
        f.restype = C.c_int
        st = f(str(path).encode(), C.byref(out), C.byref(n), C.byref(line), msg, C.c_int64(1024))
        if st == 0:
            rows = np.ctypeslib.as_array(out, shape=(n.value * 6,)).copy().reshape(-1, 6) if n.value else np.empty((0, 6))
            self._fn("free")(out)
            return rows, None
        kinds = {15: "ParseError", 16: "EmptyFile", 17: "IoError"}
        if st not in kinds:
            raise OracleError(st, "read_correspondences")
        return None, (kinds[st], msg.value.decode(), int(line.value))

    # ---- baselines (reference library only: baselines.cpp) ----------------------------------
    def grid_oracle_axis(self, z, directions=10000, eps=0.015):
        assert self.kind != "port", "baselines are checked against the compiled reference only"
        zz = np.ascontiguousarray(z, dtype=np.float64).reshape(-1, 3)
        ax = np.empty(3)
        cnt = C.c_int32()
        f = self._fn("grid_oracle_axis")
        f.restype = C.c_int
        self._ck(f(_p(zz, C.c_double), C.c_int64(zz.shape[0]), C.c_int32(directions), C.c_double(eps),
                   _p(ax, C.c_double), C.byref(cnt)), "grid_oracle_axis")
        return ax, cnt.value

    def ransac_rotation(self, corrs, iterations=1000, eps=0.015, seed=0):
        assert self.kind != "port", "baselines are checked against the compiled reference only"
        a = np.ascontiguousarray(corrs, dtype=np.float64).reshape(-1, 6)
        e = EstRef()
        f = self._fn("ransac_rotation")
        f.restype = C.c_int
        self._ck(f(_p(a, C.c_double), C.c_int64(a.shape[0]), C.c_int32(iterations), C.c_double(eps),
                   C.c_uint64(seed), C.byref(e)), "ransac_rotation")
        return self._est(e)

    # ---- solver --------------------------------------------------------------------------
    def _est(self, e):
        inl = np.ctypeslib.as_array(e.inliers, shape=(e.n_inliers,)).copy() if e.n_inliers else np.zeros(0, np.int32)
        self._fn("free")(e.inliers)
        return {"axis": np.array(e.axis[:]), "angle": e.angle, "rotation": np.array(e.rotation[:]).reshape(3, 3),
                "axis_votes": int(e.axis_votes), "inliers": inl}

    def estimate_single(self, corrs, cfg: Config | None = None):
        cfg = cfg or default_config()
        a = np.ascontiguousarray(corrs, dtype=np.float64).reshape(-1, 6)
        e = EstPort() if self.kind == "port" else EstRef()
        f = self._fn("estimate_single")
        f.restype = C.c_int
        self._ck(f(_p(a, C.c_double), C.c_int64(a.shape[0]), C.byref(cfg), C.byref(e)), "estimate_single")
        return self._est(e)

    def estimate_multi(self, corrs, cfg: Config | None = None):
        cfg = cfg or default_config()
        a = np.ascontiguousarray(corrs, dtype=np.float64).reshape(-1, 6)
        cap = max(1, cfg.max_models)
        out = ((EstPort if self.kind == "port" else EstRef) * cap)()
        nm = C.c_int32()
        f = self._fn("estimate_multi")
        f.restype = C.c_int
        st = f(_p(a, C.c_double), C.c_int64(a.shape[0]), C.byref(cfg), out, C.byref(nm))
        self._ck(st, "estimate_multi")
        return [self._est(out[k]) for k in range(min(nm.value, cap))]

    def trace(self):
        assert self.kind == "port"
        t = Trace()
        self.lib.rvo_last_trace(C.byref(t))
        return {f: (list(getattr(t, f)) if f == "start_axis" else getattr(t, f)) for f, _ in Trace._fields_}


def rotation_error_deg(r1, r2) -> float:
    c = 0.5 * (np.trace(np.asarray(r1).T @ np.asarray(r2)) - 1.0)
    return float(np.degrees(np.arccos(np.clip(c, -1.0, 1.0))))

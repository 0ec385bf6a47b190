"""rotavote-b200: B200-native spatial-voting rotation estimation (arXiv 2502.06337).

Python view of the C-ABI (include/rotavote_b200.h). The host solver is C++ inside
librotavote_b200.so; this module only marshals numpy arrays through ctypes, mirroring the
reference's public API (proj/include/rotavote/{estimator,voting,angles,geom}.hpp):
names, argument meaning, defaults and exception types are the reference's.

Arrays: correspondences (n, 6) float64 rows (x0 x1 x2 y0 y1 y2); constraints (n, 3) float64;
vote grid (G, G) uint32 indexed [iy, ix]; rotations (3, 3) float64.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, fields

import numpy as np

from . import _native, errors
from ._native import check, lib, rv_config, rv_estimate, rv_peak, rv_stage_times
from .errors import (AllDegenerate, DegenerateProjection, EmptyFile, EmptyInput, Error, InvalidConfig,  # noqa: F401
                     IoError, NoConsensus, NoPeak, NoVotes, ParseError, PoleProximity, RankDeficient)

__all__ = [
    "EstimatorConfig", "RotationEstimate", "Peak", "Context", "default_context", "errors",
    "estimate_single", "estimate_multi", "preprocess", "accumulate", "find_peaks", "blurred_argmax",
    "classify_inliers", "refine_axis", "vote_angles", "peak_angle", "peak_vote_floor", "deposit_circle_votes",
    "rodrigues", "rotation_error", "project", "unproject", "canonicalize", "orthonormal_basis",
    "correspondence_angle",
]


@dataclass
class EstimatorConfig:
    """EstimatorConfig, estimator.hpp:13-29 (same fields and defaults)."""
    grid: int = 512
    extent: float = 1.05
    theta_samples: int = 2048
    epsilon: float = 0.015
    angle_bins: int = 1024
    max_models: int = 1
    min_votes_frac: float = 0.02
    consensus_floor_mult: float = 1.5
    dedupe_overlap: float = 0.5
    tau_z: float = 1e-9
    tau_deg: float = 1e-6
    suppression_radius: int = 8
    refine: bool = True
    normalize_inputs: bool = True
    threads: int = 1

    def to_c(self) -> rv_config:
        c = rv_config()
        for f in fields(self):
            v = getattr(self, f.name)
            setattr(c, f.name, int(v) if isinstance(v, bool) else v)
        return c


@dataclass
class RotationEstimate:
    """RotationEstimate, estimator.hpp:31-38."""
    axis: np.ndarray = field(default_factory=lambda: np.array([0.0, 0.0, -1.0]))
    angle: float = 0.0
    rotation: np.ndarray = field(default_factory=lambda: np.eye(3))
    inliers: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    axis_votes: int = 0
    elapsed_s: float = 0.0


@dataclass
class Peak:
    """Peak, voting.hpp:41-46."""
    ix: int
    iy: int
    A: float
    B: float
    votes: int


def _f64(a, shape_tail) -> np.ndarray:
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.ndim == 1 and shape_tail and arr.size % shape_tail == 0:
        arr = arr.reshape(-1, shape_tail)
    return arr


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class Context:
    """One device context (stream + buffers) of the C-ABI; not thread-safe, one per thread."""

    def __init__(self, device: int = 0):
        self._lib = lib()
        h = C.c_void_p()
        check(self._lib.rv_context_create(device, C.byref(h)))
        self.handle = h

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.rv_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, st: int) -> None:
        check(st, self.handle)

    def set_stream(self, stream_ptr: int | None) -> None:
        """Run the context's work on `stream_ptr` (a cudaStream_t value, e.g. torch's
        `current_stream().cuda_stream`; 0 = the legacy default stream), or on its own stream (None)."""
        if stream_ptr is None:
            self._check(self._lib.rv_context_set_stream(self.handle, None))
        else:  # cudaStreamLegacy is the handle value 0x1 (a null handle would select the own stream)
            self._check(self._lib.rv_context_set_stream(self.handle, C.c_void_p(stream_ptr or 1)))

    def enable_timing(self, on: bool = True) -> None:
        self._check(self._lib.rv_context_enable_timing(self.handle, int(on)))

    def stage_times(self) -> dict:
        t = rv_stage_times()
        self._check(self._lib.rv_context_stage_times(self.handle, C.byref(t)))
        return {f: getattr(t, f) for f, _ in rv_stage_times._fields_}

    # ---- solver API -------------------------------------------------------------------
    def _estimate(self, e: rv_estimate, model: int) -> RotationEstimate:
        inl = np.empty(int(e.n_inliers), np.int32)
        self._check(self._lib.rv_result_inliers(self.handle, model, _ptr(inl, C.c_int32), inl.size))
        return RotationEstimate(axis=np.array(e.axis[:]), angle=e.angle,
                                rotation=np.array(e.rotation[:]).reshape(3, 3), inliers=inl,
                                axis_votes=int(e.axis_votes), elapsed_s=e.elapsed_s)

    def estimate_single(self, corrs, cfg: EstimatorConfig | None = None) -> RotationEstimate:
        """estimate_single, estimator.hpp:63-64 (host buffers: H2D + D2H inside the call)."""
        cfg = cfg or EstimatorConfig()
        a = _f64(corrs, 6)
        e = rv_estimate()
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_single(self.handle, _ptr(a, C.c_double), a.shape[0] if a.size else 0,
                                                 C.byref(c), C.byref(e)))
        return self._estimate(e, 0)

    # ---- CSV ingest (io.cpp:66-101 read_correspondences), parsed on the device ----
    def _csv(self, call) -> tuple[int, int]:
        d = C.c_void_p()
        n = C.c_int64()
        line = C.c_int64()
        st = call(d, n, line)
        if st == 15:  # ParseError carries the line
            detail = lib().rv_context_last_error(self.handle)
            raise errors.ParseError(detail.decode() if detail else "parse error", int(line.value))
        self._check(st)
        return int(d.value or 0), int(n.value)

    def parse_correspondences_device(self, text: bytes) -> tuple[int, int]:
        """CSV text -> (device pointer, rows): n x 6 f64 in context memory, valid until the next CSV
        call on this context (pass it to estimate_single_device)."""
        return self._csv(lambda d, n, l: self._lib.rv_parse_correspondences_csv(
            self.handle, text, len(text), C.byref(d), C.byref(n), C.byref(l)))

    def read_correspondences_device(self, path: str) -> tuple[int, int]:
        return self._csv(lambda d, n, l: self._lib.rv_read_correspondences_csv(
            self.handle, str(path).encode(), C.byref(d), C.byref(n), C.byref(l)))

    def _rows_to_host(self, dptr: int, n: int) -> np.ndarray:
        out = np.empty((n, 6), np.float64)
        if n:
            self._check(self._lib.rv_device_to_host(self.handle, out.ctypes.data_as(C.c_void_p), C.c_void_p(dptr),
                                                    out.nbytes))
        return out

    def read_correspondences(self, path: str) -> np.ndarray:
        """read_correspondences (io.hpp:13): n x 6 f64 [x0,x1,x2,y0,y1,y2] rows on the host."""
        d, n = self.read_correspondences_device(path)
        return self._rows_to_host(d, n)

    def parse_correspondences(self, text: bytes) -> np.ndarray:
        d, n = self.parse_correspondences_device(text)
        return self._rows_to_host(d, n)

    def estimate_single_device(self, dptr: int, n: int, cfg: EstimatorConfig | None = None) -> RotationEstimate:
        """Same solve on correspondences already resident in HBM (device pointer, n x 6 f64)."""
        cfg = cfg or EstimatorConfig()
        e = rv_estimate()
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_single_device(self.handle, C.c_void_p(dptr), n, C.byref(c), C.byref(e)))
        return self._estimate(e, 0)

    def estimate_multi(self, corrs, cfg: EstimatorConfig | None = None) -> list[RotationEstimate]:
        """estimate_multi, estimator.hpp:69-70 (sequential extraction, sorted by axis_votes)."""
        cfg = cfg or EstimatorConfig()
        a = _f64(corrs, 6)
        cap = max(1, cfg.max_models)
        out = (rv_estimate * cap)()
        nm = C.c_int32()
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_multi(self.handle, _ptr(a, C.c_double), a.shape[0] if a.size else 0,
                                                C.byref(c), out, cap, C.byref(nm)))
        return [self._estimate(out[k], k) for k in range(nm.value)]

    def estimate_multi_device(self, dptr: int, n: int, cfg: EstimatorConfig | None = None) -> list[RotationEstimate]:
        cfg = cfg or EstimatorConfig()
        cap = max(1, cfg.max_models)
        out = (rv_estimate * cap)()
        nm = C.c_int32()
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_multi_device(self.handle, C.c_void_p(dptr), n, C.byref(c), out, cap,
                                                       C.byref(nm)))
        return [self._estimate(out[k], k) for k in range(nm.value)]

    def estimate_multi_onepass(self, corrs, cfg: EstimatorConfig | None = None) -> list[RotationEstimate]:
        """EXTENSION: one vote, top-K NMS peaks, per-peak refine; no re-votes."""
        cfg = cfg or EstimatorConfig()
        a = _f64(corrs, 6)
        cap = max(1, cfg.max_models)
        out = (rv_estimate * cap)()
        nm = C.c_int32()
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_multi_onepass(self.handle, _ptr(a, C.c_double), a.shape[0] if a.size else 0,
                                                        C.byref(c), out, cap, C.byref(nm)))
        return [self._estimate(out[k], k) for k in range(nm.value)]

    def estimate_batch(self, problems, cfg: EstimatorConfig | None = None, workers: int = 0) -> list:
        """EXTENSION: estimate_single on each of many independent problems
        (a list of (n_k, 6) arrays), run concurrently on `workers` device streams. Returns one
        RotationEstimate per problem, or the RvError it raised."""
        cfg = cfg or EstimatorConfig()
        arrs = [_f64(a, 6) for a in problems]
        offs = np.zeros(len(arrs) + 1, np.int64)
        offs[1:] = np.cumsum([a.shape[0] if a.size else 0 for a in arrs])
        flat = np.ascontiguousarray(np.concatenate([a.reshape(-1, 6) for a in arrs]) if arrs else np.zeros((0, 6)))
        B = len(arrs)
        out = (rv_estimate * max(B, 1))()
        status = np.zeros(max(B, 1), np.int32)
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_batch(self.handle, _ptr(flat, C.c_double),
                                                offs.ctypes.data_as(C.POINTER(C.c_int64)), B, C.byref(c), workers,
                                                out, _ptr(status, C.c_int32)))
        res = []
        for k in range(B):
            if status[k] == 0:
                res.append(self._estimate(out[k], k))
            else:
                cls = errors.STATUS_TO_ERROR.get(int(status[k]), errors.DeviceError)
                res.append(cls(f"problem {k}: " + self._lib.rv_status_string(int(status[k])).decode()))
        return res

    # ---- baselines (reference baselines.hpp) -------------------------
    def consensus_counts(self, axes, z, epsilon: float = 0.015) -> np.ndarray:
        """consensus_count (baselines.cpp:16-24) of every axis over z, on the device."""
        a = _f64(axes, 3)
        zz = _f64(z, 3)
        out = np.zeros(a.shape[0] if a.size else 0, np.uint32)
        self._check(self._lib.rv_consensus_counts(self.handle, _ptr(a, C.c_double), out.size, _ptr(zz, C.c_double),
                                                  zz.shape[0] if zz.size else 0, epsilon,
                                                  out.ctypes.data_as(C.POINTER(C.c_uint32))))
        return out

    def grid_oracle_axis(self, z, directions: int = 10000, epsilon: float = 0.015) -> tuple[np.ndarray, int]:
        """grid_oracle_axis (baselines.hpp:38-39): best Fibonacci direction and its consensus."""
        zz = _f64(z, 3)
        ax = np.zeros(3)
        cnt = C.c_int32()
        self._check(self._lib.rv_grid_oracle_axis(self.handle, _ptr(zz, C.c_double), zz.shape[0] if zz.size else 0,
                                                  directions, epsilon, _ptr(ax, C.c_double), C.byref(cnt)))
        return ax, int(cnt.value)

    def ransac_rotation(self, corrs, iterations: int = 1000, epsilon: float = 0.015, seed: int = 0) -> RotationEstimate:
        """ransac_rotation (baselines.hpp:22-23): the reference's seeded stream, scored on the device."""
        a = _f64(corrs, 6)
        e = rv_estimate()
        self._check(self._lib.rv_ransac_rotation(self.handle, _ptr(a, C.c_double), a.shape[0] if a.size else 0,
                                                 iterations, epsilon, C.c_uint64(seed), C.byref(e)))
        return self._estimate(e, 0)

    def estimate_multi_onepass_device(self, dptr: int, n: int,
                                      cfg: EstimatorConfig | None = None) -> list[RotationEstimate]:
        cfg = cfg or EstimatorConfig()
        cap = max(1, cfg.max_models)
        out = (rv_estimate * cap)()
        nm = C.c_int32()
        c = cfg.to_c()
        self._check(self._lib.rv_estimate_multi_onepass_device(self.handle, C.c_void_p(dptr), n, C.byref(c), out, cap,
                                                               C.byref(nm)))
        return [self._estimate(out[k], k) for k in range(nm.value)]

    # ---- sharded solve (device pointers; collectives are the caller's) ----------------------
    def vote_shard(self, dptr: int, n: int, grid_dptr: int, cfg: EstimatorConfig | None = None) -> int:
        """Preprocess + vote one shard into the device grid at grid_dptr; returns kept count."""
        cfg = cfg or EstimatorConfig()
        c = cfg.to_c()
        nk = C.c_int64()
        self._check(self._lib.rv_vote_shard(self.handle, C.c_void_p(dptr), n, C.byref(c), C.c_void_p(grid_dptr),
                                            C.byref(nk)))
        return nk.value

    def estimate_single_prevoted(self, dptr: int, n: int, grid_dptr: int,
                                 cfg: EstimatorConfig | None = None) -> RotationEstimate:
        cfg = cfg or EstimatorConfig()
        c = cfg.to_c()
        e = rv_estimate()
        self._check(self._lib.rv_estimate_single_prevoted(self.handle, C.c_void_p(dptr), n, C.byref(c),
                                                          C.c_void_p(grid_dptr), C.byref(e)))
        return self._estimate(e, 0)

    # ---- sharded finish steps (include/rotavote_b200.h) ------------------
    def peak_start_axis(self, grid_dptr: int, cfg: EstimatorConfig | None = None):
        """find_peaks(K=1) + estimate_from_peak's start axis from a device grid -> (axis, votes, total)."""
        c = (cfg or EstimatorConfig()).to_c()
        axis = np.zeros(3)
        votes, total = C.c_uint32(), C.c_uint64()
        self._check(self._lib.rv_peak_start_axis(self.handle, C.c_void_p(grid_dptr), C.byref(c),
                                                 _ptr(axis, C.c_double), C.byref(votes), C.byref(total)))
        return axis, votes.value, total.value

    def shard_classify(self, axis, epsilon: float, slot: int, compare_prev: bool):
        """classify this context's shard into bitmask `slot` -> (count, scatter[6], differs)."""
        a = np.ascontiguousarray(axis, dtype=np.float64)
        cnt, diff = C.c_int64(), C.c_int32()
        sc = np.zeros(6)
        self._check(self._lib.rv_shard_classify(self.handle, _ptr(a, C.c_double), epsilon, slot, int(compare_prev),
                                                C.byref(cnt), _ptr(sc, C.c_double), C.byref(diff)))
        return cnt.value, sc, bool(diff.value)

    def shard_refine(self, axis0, cfg: EstimatorConfig | None = None, n_dev: int = 1, rank: int = 0,
                     lines=None, epoch: int = 0):
        """refine_loop of this context's shard as one device-resident loop; with n_dev > 1 the
        per-pass partials are exchanged with the other devices through `lines` (every rank's line
        buffer, rank order: rv_shard_lines_export / rv_shard_lines_open) ->
        (axis, count, local_count, scatter[6], refits); final set in slot 0."""
        c = (cfg or EstimatorConfig()).to_c()
        a0 = np.ascontiguousarray(axis0, dtype=np.float64)
        ax, sc = np.zeros(3), np.zeros(6)
        cnt, loc, rf = C.c_int64(), C.c_int64(), C.c_int32()
        arr = (C.c_void_p * max(1, n_dev))(*(lines or [])) if n_dev > 1 else None
        self._check(self._lib.rv_shard_refine(self.handle, _ptr(a0, C.c_double), C.byref(c), n_dev, rank, arr, epoch,
                                              _ptr(ax, C.c_double), C.byref(cnt), C.byref(loc), _ptr(sc, C.c_double),
                                              C.byref(rf)))
        return ax, cnt.value, loc.value, sc, rf.value

    def shard_lines_export(self) -> tuple[int, bytes]:
        """this context's line buffer for a cross-process shard_refine -> (device pointer, IPC handle)."""
        ptr = C.c_void_p()
        h = C.create_string_buffer(64)
        self._check(self._lib.rv_shard_lines_export(self.handle, C.byref(ptr), h))
        return ptr.value, h.raw

    def shard_lines_open(self, handle: bytes) -> int:
        """map a peer rank's line buffer from its IPC handle -> device pointer (closed with the context)."""
        ptr = C.c_void_p()
        self._check(self._lib.rv_shard_lines_open(self.handle, C.create_string_buffer(handle, 64), C.byref(ptr)))
        return ptr.value

    def shard_inliers(self, slot: int, offset: int, count: int) -> np.ndarray:
        out = np.zeros(max(count, 1), np.int32)
        got = C.c_int64()
        self._check(self._lib.rv_shard_inliers(self.handle, slot, offset, _ptr(out, C.c_int32), count, C.byref(got)))
        return out[:got.value]

    def shard_angle_hist(self, axis, cfg: EstimatorConfig | None = None):
        cfg = cfg or EstimatorConfig()
        c = cfg.to_c()
        a = np.ascontiguousarray(axis, dtype=np.float64)
        bins = np.zeros(cfg.angle_bins, np.uint32)
        contrib = C.c_uint64()
        self._check(self._lib.rv_shard_angle_hist(self.handle, _ptr(a, C.c_double), C.byref(c),
                                                  _ptr(bins, C.c_uint32), C.byref(contrib)))
        return bins, contrib.value

    def shard_angle_sums(self, bins_total, cfg: EstimatorConfig | None = None) -> np.ndarray:
        c = (cfg or EstimatorConfig()).to_c()
        b = np.ascontiguousarray(bins_total, dtype=np.uint32)
        sums = np.zeros(2)
        self._check(self._lib.rv_shard_angle_sums(self.handle, _ptr(b, C.c_uint32), C.byref(c),
                                                  _ptr(sums, C.c_double)))
        return sums

    # ---- path functions -----------------------------------------------------------------
    def preprocess(self, corrs, tau_z: float = 1e-9, normalize: bool = True):
        """preprocess, estimator.hpp:47-48 -> (constraints (k,3), kept (k,), dropped (d,))."""
        a = _f64(corrs, 6)
        n = a.shape[0] if a.size else 0
        z = np.empty((max(n, 1), 3))
        kept = np.empty(max(n, 1), np.int32)
        dropped = np.empty(max(n, 1), np.int32)
        nk, nd = C.c_int64(), C.c_int64()
        self._check(self._lib.rv_preprocess(self.handle, _ptr(a, C.c_double), n, tau_z, int(normalize),
                                            _ptr(z, C.c_double), _ptr(kept, C.c_int32), _ptr(dropped, C.c_int32),
                                            C.byref(nk), C.byref(nd)))
        return z[:nk.value].copy(), kept[:nk.value].copy(), dropped[:nd.value].copy()

    def accumulate(self, constraints, grid: int = 512, extent: float = 1.05, samples: int = 2048,
                   threads: int = 1) -> np.ndarray:
        """accumulate, voting.hpp:64-65 -> (grid, grid) uint32 counts[iy, ix]."""
        z = _f64(constraints, 3)
        n = z.shape[0] if z.size else 0
        out = np.empty((max(grid, 1), max(grid, 1)), np.uint32)
        self._check(self._lib.rv_accumulate(self.handle, _ptr(z, C.c_double), n, grid, extent, samples,
                                            _ptr(out, C.c_uint32)))
        return out

    def deposit_circle_votes(self, z, counts: np.ndarray, extent: float = 1.05, samples: int = 2048) -> None:
        """deposit_circle_votes, voting.hpp:60 (in-place on a (G, G) uint32 grid)."""
        zz = _f64(z, 0).reshape(3)
        assert counts.dtype == np.uint32 and counts.flags.c_contiguous
        self._check(self._lib.rv_deposit_circle_votes(self.handle, _ptr(zz, C.c_double), _ptr(counts, C.c_uint32),
                                                      counts.shape[0], extent, samples))

    def find_peaks(self, counts: np.ndarray, max_peaks: int, suppression_radius: int, min_votes: int,
                   extent: float = 1.05) -> list[Peak]:
        """find_peaks, voting.hpp:70-71."""
        g = np.ascontiguousarray(counts, dtype=np.uint32)
        out = (rv_peak * max(1, max_peaks))()
        n = C.c_int32()
        self._check(self._lib.rv_find_peaks(self.handle, _ptr(g, C.c_uint32), g.shape[0], extent, max_peaks,
                                            suppression_radius, min_votes, out, C.byref(n)))
        return [Peak(out[k].ix, out[k].iy, out[k].A, out[k].B, out[k].votes) for k in range(n.value)]

    def blurred_argmax(self, counts: np.ndarray, radius: int, extent: float = 1.05) -> Peak:
        """blurred_argmax, voting.hpp:80."""
        g = np.ascontiguousarray(counts, dtype=np.uint32)
        p = rv_peak()
        self._check(self._lib.rv_blurred_argmax(self.handle, _ptr(g, C.c_uint32), g.shape[0], extent, radius,
                                                C.byref(p)))
        return Peak(p.ix, p.iy, p.A, p.B, p.votes)

    def classify_inliers(self, axis, constraints, epsilon: float) -> np.ndarray:
        """classify_inliers, estimator.hpp:51-52."""
        ax = _f64(axis, 0).reshape(3)
        z = _f64(constraints, 3)
        n = z.shape[0] if z.size else 0
        out = np.empty(max(n, 1), np.int32)
        m = C.c_int64()
        self._check(self._lib.rv_classify_inliers(self.handle, _ptr(ax, C.c_double), _ptr(z, C.c_double), n, epsilon,
                                                  _ptr(out, C.c_int32), C.byref(m)))
        return out[:m.value].copy()

    def refine_axis(self, constraints) -> np.ndarray:
        """refine_axis, estimator.hpp:57."""
        z = _f64(constraints, 3)
        n = z.shape[0] if z.size else 0
        out = np.empty(3)
        self._check(self._lib.rv_refine_axis(self.handle, _ptr(z, C.c_double), n, _ptr(out, C.c_double)))
        return out

    def vote_angles(self, axis, corrs, indices, bin_count: int, tau: float = 1e-6):
        """vote_angles, angles.hpp:37-40 -> dict(bins, contributing, degenerate, raw_angles)."""
        ax = _f64(axis, 0).reshape(3)
        a = _f64(corrs, 6)
        idx = np.ascontiguousarray(np.asarray(indices, dtype=np.int32))
        bins = np.empty(max(bin_count, 1), np.uint32)
        raw = np.empty(max(idx.size, 1))
        contrib, degen = C.c_uint64(), C.c_uint64()
        self._check(self._lib.rv_vote_angles(self.handle, _ptr(ax, C.c_double), _ptr(a, C.c_double),
                                             a.shape[0] if a.size else 0, _ptr(idx, C.c_int32), idx.size, bin_count,
                                             tau, _ptr(bins, C.c_uint32), C.byref(contrib), C.byref(degen),
                                             _ptr(raw, C.c_double)))
        return {"bins": bins[:bin_count], "contributing": contrib.value, "degenerate": degen.value,
                "raw_angles": raw[:contrib.value].copy()}

    def peak_angle(self, hist: dict, refine: bool, raw_angles=None) -> float:
        """peak_angle, angles.hpp:44-49."""
        bins = np.ascontiguousarray(hist["bins"], dtype=np.uint32)
        raw = _f64(hist["raw_angles"] if raw_angles is None else raw_angles, 0).reshape(-1)
        out = C.c_double()
        self._check(self._lib.rv_peak_angle(self.handle, _ptr(bins, C.c_uint32), bins.size, hist["contributing"],
                                            int(refine), _ptr(raw, C.c_double), raw.size, C.byref(out)))
        return out.value


_default: Context | None = None


def axis_from_scatter(scatter) -> np.ndarray:
    """refine_axis's 3x3 eigen-solve (estimator.cpp:299-309) of a summed scatter (xx xy xz yy yz zz)."""
    sc = np.ascontiguousarray(scatter, dtype=np.float64)
    axis = np.zeros(3)
    st = _native.lib().rv_axis_from_scatter(_ptr(sc, C.c_double), _ptr(axis, C.c_double))
    _native.check(st)
    return axis


class MultiContext:
    """Several B200s in one process (rv_multi_*): NCCL clique, sharded estimate_single / accumulate."""

    def __init__(self, devices):
        self._lib = _native.lib()
        devs = np.ascontiguousarray(list(devices), dtype=np.int32)
        h = C.c_void_p()
        st = self._lib.rv_multi_create(_ptr(devs, C.c_int32), len(devs), C.byref(h))
        _native.check(st)
        self.handle = h
        self.devices = list(devs)

    def close(self) -> None:
        if getattr(self, "handle", None):
            self._lib.rv_multi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def nccl_version(self) -> int:
        return self._lib.rv_multi_nccl_version(self.handle)

    def _check(self, st: int) -> None:
        if st != 0:
            cls = errors.STATUS_TO_ERROR.get(st, errors.DeviceError)
            raise cls(self._lib.rv_status_string(st).decode() + ": " + self._lib.rv_multi_last_error(self.handle).decode())

    def estimate_single(self, corrs, cfg: EstimatorConfig | None = None) -> RotationEstimate:
        a = _f64(corrs, 6)
        c = (cfg or EstimatorConfig()).to_c()
        e = rv_estimate()
        self._check(self._lib.rv_multi_estimate_single(self.handle, _ptr(a, C.c_double), a.shape[0], C.byref(c),
                                                       C.byref(e)))
        inl = np.zeros(max(e.n_inliers, 1), np.int32)
        self._check(self._lib.rv_multi_result_inliers(self.handle, _ptr(inl, C.c_int32), e.n_inliers))
        return RotationEstimate(axis=np.array(e.axis[:]), angle=e.angle, rotation=np.array(e.rotation[:]).reshape(3, 3),
                                inliers=inl[:e.n_inliers], axis_votes=int(e.axis_votes), elapsed_s=e.elapsed_s)

    def accumulate(self, constraints, grid: int = 512, extent: float = 1.05, samples: int = 2048) -> np.ndarray:
        z = _f64(constraints, 3)
        out = np.zeros((grid, grid), np.uint32)
        self._check(self._lib.rv_multi_accumulate(self.handle, _ptr(z, C.c_double), z.shape[0], grid, extent, samples,
                                                  _ptr(out, C.c_uint32)))
        return out


def default_context() -> Context:
    global _default
    if _default is None:
        _default = Context(0)
    return _default


def estimate_single(corrs, cfg: EstimatorConfig | None = None) -> RotationEstimate:
    return default_context().estimate_single(corrs, cfg)


def estimate_multi(corrs, cfg: EstimatorConfig | None = None) -> list[RotationEstimate]:
    return default_context().estimate_multi(corrs, cfg)


def preprocess(corrs, tau_z: float = 1e-9, normalize: bool = True):
    return default_context().preprocess(corrs, tau_z, normalize)


def accumulate(constraints, grid: int = 512, extent: float = 1.05, samples: int = 2048, threads: int = 1):
    return default_context().accumulate(constraints, grid, extent, samples, threads)


def deposit_circle_votes(z, counts, extent: float = 1.05, samples: int = 2048):
    return default_context().deposit_circle_votes(z, counts, extent, samples)


def find_peaks(counts, max_peaks, suppression_radius, min_votes, extent: float = 1.05):
    return default_context().find_peaks(counts, max_peaks, suppression_radius, min_votes, extent)


def blurred_argmax(counts, radius, extent: float = 1.05):
    return default_context().blurred_argmax(counts, radius, extent)


def classify_inliers(axis, constraints, epsilon):
    return default_context().classify_inliers(axis, constraints, epsilon)


def refine_axis(constraints):
    return default_context().refine_axis(constraints)


def vote_angles(axis, corrs, indices, bin_count, tau: float = 1e-6):
    return default_context().vote_angles(axis, corrs, indices, bin_count, tau)


def peak_angle(hist, refine, raw_angles=None):
    return default_context().peak_angle(hist, refine, raw_angles)


def peak_vote_floor(cfg: EstimatorConfig, n_constraints: int) -> int:
    c = cfg.to_c()
    return int(lib().rv_peak_vote_floor(C.byref(c), n_constraints))


# ---- geometry (geom.hpp:25-43; host arithmetic in the library) -----------------------------
def rodrigues(axis, angle: float) -> np.ndarray:
    ax = _f64(axis, 0).reshape(3)
    r = np.empty(9)
    lib().rv_rodrigues(_ptr(ax, C.c_double), angle, _ptr(r, C.c_double))
    return r.reshape(3, 3)


def rotation_error(r_gt, r_opt) -> float:
    a = np.ascontiguousarray(r_gt, dtype=np.float64).reshape(9)
    b = np.ascontiguousarray(r_opt, dtype=np.float64).reshape(9)
    return float(lib().rv_rotation_error(_ptr(a, C.c_double), _ptr(b, C.c_double)))


def project(p):
    pp = _f64(p, 0).reshape(3)
    A, B = C.c_double(), C.c_double()
    check(lib().rv_project(_ptr(pp, C.c_double), C.byref(A), C.byref(B)))
    return A.value, B.value


def unproject(A: float, B: float) -> np.ndarray:
    o = np.empty(3)
    lib().rv_unproject(A, B, _ptr(o, C.c_double))
    return o


def canonicalize(p) -> np.ndarray:
    pp = _f64(p, 0).reshape(3)
    o = np.empty(3)
    lib().rv_canonicalize(_ptr(pp, C.c_double), _ptr(o, C.c_double))
    return o


def orthonormal_basis(z):
    zz = _f64(z, 0).reshape(3)
    a1, a2 = np.empty(3), np.empty(3)
    lib().rv_orthonormal_basis(_ptr(zz, C.c_double), _ptr(a1, C.c_double), _ptr(a2, C.c_double))
    return a1, a2


def correspondence_angle(axis, x, y, tau: float = 1e-6) -> float:
    a, xx, yy = (_f64(v, 0).reshape(3) for v in (axis, x, y))
    out = C.c_double()
    check(lib().rv_correspondence_angle(_ptr(a, C.c_double), _ptr(xx, C.c_double), _ptr(yy, C.c_double), tau,
                                        C.byref(out)))
    return out.value

"""ctypes binding of the C-ABI in include/rotavote_b200.h (librotavote_b200.so, sm_100a).

The library is built in-tree by paper_2502_06337_b200/build.py. There is no CPU fallback:
if the shared library is missing, loading fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

from . import errors

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "librotavote_b200.so"
# dev A/B of kernel variants only (tools/ab_vote.py): another in-tree build of the same library
if os.environ.get("RV_LIB_PATH"):
    LIB_PATH = Path(os.environ["RV_LIB_PATH"]).resolve()

c_double_p = C.POINTER(C.c_double)
c_int32_p = C.POINTER(C.c_int32)
c_uint32_p = C.POINTER(C.c_uint32)
c_int64_p = C.POINTER(C.c_int64)
c_uint64_p = C.POINTER(C.c_uint64)


class rv_config(C.Structure):
    _fields_ = [
        ("grid", C.c_int32),
        ("extent", C.c_double),
        ("theta_samples", C.c_int32),
        ("epsilon", C.c_double),
        ("angle_bins", C.c_int32),
        ("max_models", C.c_int32),
        ("min_votes_frac", C.c_double),
        ("consensus_floor_mult", C.c_double),
        ("dedupe_overlap", C.c_double),
        ("tau_z", C.c_double),
        ("tau_deg", C.c_double),
        ("suppression_radius", C.c_int32),
        ("refine", C.c_int32),
        ("normalize_inputs", C.c_int32),
        ("threads", C.c_int32),
    ]


class rv_peak(C.Structure):
    _fields_ = [("ix", C.c_int32), ("iy", C.c_int32), ("A", C.c_double), ("B", C.c_double), ("votes", C.c_uint32)]


class rv_estimate(C.Structure):
    _fields_ = [
        ("axis", C.c_double * 3),
        ("angle", C.c_double),
        ("rotation", C.c_double * 9),
        ("axis_votes", C.c_uint32),
        ("n_inliers", C.c_int64),
        ("elapsed_s", C.c_double),
    ]


class rv_stage_times(C.Structure):
    _fields_ = [
        ("preprocess_ms", C.c_double),
        ("vote_ms", C.c_double),
        ("peaks_ms", C.c_double),
        ("refine_ms", C.c_double),
        ("angles_ms", C.c_double),
        ("total_ms", C.c_double),
        ("vote_pairs", C.c_int64),
        ("vote_fallback_pairs", C.c_int64),
        ("vote_guard_reruns", C.c_int64),
        ("vote_samples", C.c_int64),
        ("vote_launches", C.c_int32),
        ("kernel_launches", C.c_int32),
        ("vote_kernel_ms", C.c_double),
        ("csv_host_fields", C.c_int64),
    ]


_lib = None

# (name, restype, argtypes)
_SIGS = [
    ("rv_abi_version", C.c_int32, []),
    ("rv_config_default", None, [C.POINTER(rv_config)]),
    ("rv_status_string", C.c_char_p, [C.c_int]),
    ("rv_context_create", C.c_int, [C.c_int32, C.POINTER(C.c_void_p)]),
    ("rv_context_destroy", None, [C.c_void_p]),
    ("rv_context_set_stream", C.c_int, [C.c_void_p, C.c_void_p]),
    ("rv_context_last_error", C.c_char_p, [C.c_void_p]),
    ("rv_context_enable_timing", C.c_int, [C.c_void_p, C.c_int32]),
    ("rv_context_stage_times", C.c_int, [C.c_void_p, C.POINTER(rv_stage_times)]),
    ("rv_estimate_single", C.c_int, [C.c_void_p, c_double_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate)]),
    ("rv_estimate_single_device", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate)]),
    ("rv_estimate_multi", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate), C.c_int32, c_int32_p]),
    ("rv_estimate_multi_device", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate), C.c_int32, c_int32_p]),
    ("rv_estimate_multi_onepass", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate), C.c_int32, c_int32_p]),
    ("rv_estimate_multi_onepass_device", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate), C.c_int32, c_int32_p]),
    ("rv_estimate_batch", C.c_int,
     [C.c_void_p, c_double_p, C.POINTER(C.c_int64), C.c_int32, C.POINTER(rv_config), C.c_int32,
      C.POINTER(rv_estimate), c_int32_p]),
    ("rv_consensus_counts", C.c_int,
     [C.c_void_p, c_double_p, C.c_int32, c_double_p, C.c_int64, C.c_double, C.POINTER(C.c_uint32)]),
    ("rv_grid_oracle_axis", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.c_int32, C.c_double, c_double_p, c_int32_p]),
    ("rv_ransac_rotation", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.c_int32, C.c_double, C.c_uint64, C.POINTER(rv_estimate)]),
    ("rv_result_inliers", C.c_int, [C.c_void_p, C.c_int32, c_int32_p, C.c_int64]),
    ("rv_vote_shard", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(rv_config), C.c_void_p, c_int64_p]),
    ("rv_estimate_single_prevoted", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.POINTER(rv_config), C.c_void_p, C.POINTER(rv_estimate)]),
    ("rv_peak_start_axis", C.c_int,
     [C.c_void_p, C.c_void_p, C.POINTER(rv_config), c_double_p, C.POINTER(C.c_uint32), c_uint64_p]),
    ("rv_shard_classify", C.c_int,
     [C.c_void_p, c_double_p, C.c_double, C.c_int32, C.c_int32, c_int64_p, c_double_p, c_int32_p]),
    ("rv_axis_from_scatter", C.c_int, [c_double_p, c_double_p]),
    ("rv_shard_refine", C.c_int,
     [C.c_void_p, c_double_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p, C.c_uint64, c_double_p, c_int64_p,
      c_int64_p, c_double_p, c_int32_p]),
    ("rv_shard_lines_export", C.c_int, [C.c_void_p, C.POINTER(C.c_void_p), C.c_char_p]),
    ("rv_shard_lines_open", C.c_int, [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p)]),
    ("rv_shard_inliers", C.c_int, [C.c_void_p, C.c_int32, C.c_int64, c_int32_p, C.c_int64, c_int64_p]),
    ("rv_shard_angle_hist", C.c_int, [C.c_void_p, c_double_p, C.POINTER(rv_config), c_uint32_p, c_uint64_p]),
    ("rv_shard_angle_sums", C.c_int, [C.c_void_p, c_uint32_p, C.POINTER(rv_config), c_double_p]),
    ("rv_multi_create", C.c_int, [c_int32_p, C.c_int32, C.POINTER(C.c_void_p)]),
    ("rv_multi_destroy", None, [C.c_void_p]),
    ("rv_multi_size", C.c_int32, [C.c_void_p]),
    ("rv_multi_last_error", C.c_char_p, [C.c_void_p]),
    ("rv_multi_nccl_version", C.c_int32, [C.c_void_p]),
    ("rv_multi_estimate_single", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.POINTER(rv_config), C.POINTER(rv_estimate)]),
    ("rv_multi_result_inliers", C.c_int, [C.c_void_p, c_int32_p, C.c_int64]),
    ("rv_multi_accumulate", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.c_int32, C.c_double, C.c_int32, c_uint32_p]),
    ("rv_preprocess", C.c_int,
     [C.c_void_p, c_double_p, C.c_int64, C.c_double, C.c_int32, c_double_p, c_int32_p, c_int32_p, c_int64_p, c_int64_p]),
    ("rv_accumulate", C.c_int, [C.c_void_p, c_double_p, C.c_int64, C.c_int32, C.c_double, C.c_int32, c_uint32_p]),
    ("rv_accumulate_device", C.c_int,
     [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_double, C.c_int32, C.c_void_p]),
    ("rv_deposit_circle_votes", C.c_int, [C.c_void_p, c_double_p, c_uint32_p, C.c_int32, C.c_double, C.c_int32]),
    ("rv_find_peaks", C.c_int,
     [C.c_void_p, c_uint32_p, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_uint32, C.POINTER(rv_peak), c_int32_p]),
    ("rv_blurred_argmax", C.c_int, [C.c_void_p, c_uint32_p, C.c_int32, C.c_double, C.c_int32, C.POINTER(rv_peak)]),
    ("rv_classify_inliers", C.c_int, [C.c_void_p, c_double_p, c_double_p, C.c_int64, C.c_double, c_int32_p, c_int64_p]),
    ("rv_refine_axis", C.c_int, [C.c_void_p, c_double_p, C.c_int64, c_double_p]),
    ("rv_vote_angles", C.c_int,
     [C.c_void_p, c_double_p, c_double_p, C.c_int64, c_int32_p, C.c_int64, C.c_int32, C.c_double, c_uint32_p,
      c_uint64_p, c_uint64_p, c_double_p]),
    ("rv_peak_angle", C.c_int,
     [C.c_void_p, c_uint32_p, C.c_int32, C.c_uint64, C.c_int32, c_double_p, C.c_int64, c_double_p]),
    ("rv_peak_vote_floor", C.c_uint32, [C.POINTER(rv_config), C.c_int64]),
    ("rv_parse_correspondences_csv", C.c_int,
     [C.c_void_p, C.c_char_p, C.c_int64, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("rv_read_correspondences_csv", C.c_int,
     [C.c_void_p, C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("rv_device_to_host", C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64]),
    ("rv_rodrigues", None, [c_double_p, C.c_double, c_double_p]),
    ("rv_rotation_error", C.c_double, [c_double_p, c_double_p]),
    ("rv_project", C.c_int, [c_double_p, c_double_p, c_double_p]),
    ("rv_unproject", None, [C.c_double, C.c_double, c_double_p]),
    ("rv_canonicalize", None, [c_double_p, c_double_p]),
    ("rv_orthonormal_basis", None, [c_double_p, c_double_p, c_double_p]),
    ("rv_correspondence_angle", C.c_int, [c_double_p, c_double_p, c_double_p, C.c_double, c_double_p]),
]

EXPORTED_SYMBOLS = [name for name, _, _ in _SIGS]


def lib() -> C.CDLL:
    """Loads librotavote_b200.so (raises if it has not been built: no CPU fallback)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build the sm_100a library first "
                "(python paper_2502_06337_b200/build.py or __graft_entry__.build())")
        handle = C.CDLL(str(LIB_PATH))
        for name, res, args in _SIGS:
            fn = getattr(handle, name)
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def check(status: int, ctx=None) -> None:
    if status == 0:
        return
    cls = errors.STATUS_TO_ERROR.get(status, errors.DeviceError)
    msg = lib().rv_status_string(status).decode()
    if ctx is not None:
        detail = lib().rv_context_last_error(ctx)
        if detail:
            msg += ": " + detail.decode()
    raise cls(msg)

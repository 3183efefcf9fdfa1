"""ctypes binding of libfht.so (include/fht.h). Argument marshalling only.

The structures below mirror include/fht.h field by field. Nothing here computes any part of
the transform: every step runs in the CUDA kernels behind the C ABI. If the shared library
is missing this module raises at import time -- there is no fallback path.
"""
from __future__ import annotations

import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# FHT_LIB overrides the library path (A/B timing of alternative builds, tools/abbench.py)
LIB_PATH = os.environ.get("FHT_LIB") or os.path.join(_HERE, "libfht.so")

FHT_U8, FHT_I32, FHT_F32 = 0, 1, 2
FHT_QA, FHT_QB, FHT_QC, FHT_QD = 0, 1, 2, 3
FHT_MODE_QUADRANT, FHT_MODE_FULL, FHT_MODE_RANGE = 0, 1, 2
FHT_LAYOUT_QUADS, FHT_LAYOUT_CONCAT = 0, 1

FHT_PLAN_PRUNED, FHT_PLAN_HORIZONTAL = 1, 2

STATUS = {
    0: "FHT_OK", -1: "FHT_ERR_ARG", -2: "FHT_ERR_DTYPE", -3: "FHT_ERR_SHAPE", -4: "FHT_ERR_ALIGN",
    -5: "FHT_ERR_UNSUPPORTED", -6: "FHT_ERR_WORKSPACE", -7: "FHT_ERR_STATE", -8: "FHT_ERR_CUDA",
}

EXPORTED = (
    "fht_hough_describe", "fht_workspace_bytes", "fht_quadrant", "fht_full", "fht_angle_plan", "fht_angle_of_row",
    "fht_angle_plan_make_pruned", "fht_angle_plan_make_ex", "fht_angle_range", "fht_angle_range_workspace_bytes",
    "fht_angle_range_plan", "fhtshift", "fht_status_string", "fht_peaks_workspace_bytes",
    "fht_peaks", "fht_cell_segment", "fht_hough_describe_pad", "fht_quadrant_workspace_bytes",
    "fht_shard_describe", "fht_shard_pass1", "fht_shard_pass2",
)


class FhtImage(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("_pad0", ctypes.c_int32),
        ("batch", ctypes.c_int64), ("h", ctypes.c_int64), ("w", ctypes.c_int64),
        ("batch_stride", ctypes.c_int64), ("row_stride", ctypes.c_int64),
    ]


class FhtAnglePlan(ctypes.Structure):
    _fields_ = [
        ("theta_min_deg", ctypes.c_double), ("theta_max_deg", ctypes.c_double),
        ("k_lo", ctypes.c_double), ("k_hi", ctypes.c_double), ("alpha", ctypes.c_double), ("g", ctypes.c_double),
        ("h", ctypes.c_int64), ("w", ctypes.c_int64), ("Hp", ctypes.c_int64),
        ("w_content", ctypes.c_int64), ("W", ctypes.c_int64), ("e_min", ctypes.c_int64), ("e_max", ctypes.c_int64),
        ("rows", ctypes.c_int64), ("transposed", ctypes.c_int64),
    ]


class FhtSegment(ctypes.Structure):
    _fields_ = [
        ("quadrant", ctypes.c_int32), ("s", ctypes.c_int32), ("npix", ctypes.c_int64),
        ("x0", ctypes.c_int64), ("y0", ctypes.c_int64), ("x1", ctypes.c_int64), ("y1", ctypes.c_int64),
    ]


class FhtHough(ctypes.Structure):
    _fields_ = [
        ("data", ctypes.c_void_p), ("dtype", ctypes.c_int32), ("mode", ctypes.c_int32),
        ("layout", ctypes.c_int32), ("shifted", ctypes.c_int32), ("quadrant", ctypes.c_int32),
        ("_pad0", ctypes.c_int32),
        ("batch", ctypes.c_int64), ("nquad", ctypes.c_int64), ("rows", ctypes.c_int64), ("cols", ctypes.c_int64),
        ("batch_stride", ctypes.c_int64), ("quad_stride", ctypes.c_int64), ("row_stride", ctypes.c_int64),
        ("h", ctypes.c_int64), ("w", ctypes.c_int64), ("Hp", ctypes.c_int64), ("Wp", ctypes.c_int64),
        ("plan", FhtAnglePlan), ("row0", ctypes.c_int64),
    ]


class FhtShard(ctypes.Structure):
    _fields_ = [
        ("world", ctypes.c_int32), ("rank", ctypes.c_int32), ("m", ctypes.c_int32), ("L", ctypes.c_int32),
        ("S", ctypes.c_int64), ("J", ctypes.c_int64), ("rows_per_rank", ctypes.c_int64), ("pitch", ctypes.c_int64),
        ("scratch_es", ctypes.c_int32), ("_pad0", ctypes.c_int32), ("chunk_rows", ctypes.c_int64),
        ("chunk_bytes", ctypes.c_int64), ("send_bytes", ctypes.c_int64), ("recv_bytes", ctypes.c_int64),
        ("band", FhtHough),
    ]


class FhtExecOpts(ctypes.Structure):
    _fields_ = [("events", ctypes.POINTER(ctypes.c_void_p)), ("n_events", ctypes.c_int32), ("_pad0", ctypes.c_int32),
                ("aux_stream", ctypes.c_void_p)]


class FhtError(RuntimeError):
    def __init__(self, fn: str, status: int):
        super().__init__(f"{fn} failed: {STATUS.get(status, status)}")
        self.status = status


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
    lib = ctypes.CDLL(LIB_PATH)
    P = ctypes.POINTER
    vp, i64, i32, sz, dbl = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t, ctypes.c_double
    lib.fht_hough_describe.argtypes = [i32, i32, i32, P(FhtImage), P(FhtAnglePlan), P(FhtHough)]
    lib.fht_workspace_bytes.argtypes = [i32, P(FhtImage), P(FhtAnglePlan)]
    lib.fht_workspace_bytes.restype = sz
    lib.fht_quadrant.argtypes = [P(FhtImage), i32, i64, P(FhtHough), P(FhtHough), vp, sz, vp, P(FhtExecOpts)]
    lib.fht_full.argtypes = [P(FhtImage), i32, P(FhtHough), P(FhtHough), vp, sz, vp, P(FhtExecOpts)]
    lib.fht_angle_plan.argtypes = [i64, i64, dbl, dbl, P(FhtAnglePlan)]
    lib.fht_angle_of_row.argtypes = [P(FhtAnglePlan), i64, P(dbl)]
    lib.fht_angle_plan_make_pruned.argtypes = [i64, i64, dbl, dbl, P(FhtAnglePlan)]
    lib.fht_angle_plan_make_ex.argtypes = [i64, i64, dbl, dbl, i32, P(FhtAnglePlan)]
    lib.fht_angle_range.argtypes = [P(FhtImage), dbl, dbl, P(FhtHough), P(FhtHough), vp, sz, vp, P(FhtExecOpts)]
    lib.fht_angle_range_workspace_bytes.argtypes = [P(FhtImage), dbl, dbl]
    lib.fht_angle_range_workspace_bytes.restype = sz
    lib.fht_angle_range_plan.argtypes = [P(FhtImage), P(FhtAnglePlan), P(FhtHough), P(FhtHough), vp, sz, vp,
                                         P(FhtExecOpts)]
    lib.fhtshift.argtypes = [P(FhtHough), P(FhtHough), vp]
    lib.fht_peaks_workspace_bytes.argtypes = [P(FhtHough)]
    lib.fht_peaks_workspace_bytes.restype = sz
    lib.fht_peaks.argtypes = [P(FhtHough), i32, vp, vp, vp, vp, sz, vp]
    lib.fht_cell_segment.argtypes = [P(FhtHough), i64, i64, i64, P(FhtSegment)]
    lib.fht_hough_describe_pad.argtypes = [i32, P(FhtImage), i64, P(FhtHough)]
    lib.fht_quadrant_workspace_bytes.argtypes = [P(FhtImage), i32, i64]
    lib.fht_quadrant_workspace_bytes.restype = sz
    lib.fht_shard_describe.argtypes = [P(FhtImage), i32, i32, P(FhtShard)]
    lib.fht_shard_pass1.argtypes = [P(FhtImage), P(FhtShard), P(vp), vp]
    lib.fht_shard_pass2.argtypes = [P(FhtImage), P(FhtShard), vp, P(FhtHough), P(FhtHough), vp]
    lib.fht_status_string.argtypes = [i32]
    lib.fht_status_string.restype = ctypes.c_char_p
    for name in ("fht_hough_describe", "fht_quadrant", "fht_full", "fht_angle_plan", "fht_angle_of_row",
                 "fht_angle_plan_make_pruned", "fht_angle_plan_make_ex", "fht_angle_range", "fht_angle_range_plan",
                 "fhtshift", "fht_peaks", "fht_cell_segment", "fht_hough_describe_pad", "fht_shard_describe",
                 "fht_shard_pass1", "fht_shard_pass2"):
        getattr(lib, name).restype = i32
    return lib


lib = _load()


def check(fn: str, status: int) -> int:
    if status < 0:
        raise FhtError(fn, status)
    return status

"""ctypes mirrors of the structs in include/trb.h (the C-ABI boundary)."""
from __future__ import annotations

import ctypes as C

import numpy as np


class MOTION_CFG(C.Structure):
    """trb_motion_config == MotionConfig (motion.hpp:44-56) + morph extension."""
    _fields_ = [("method", C.c_int32), ("window", C.c_int32), ("threshold", C.c_int32), ("bins", C.c_int32),
                ("warp", C.c_int32), ("morph", C.c_int32)]

    def __init__(self, method=0, window=91, threshold=25, bins=32, warp=0, morph=0):
        super().__init__(method, window, threshold, bins, warp, morph)


class SEG_CFG(C.Structure):
    """trb_seg_config == SegmentationConfig (segmentation.hpp:25-34)."""
    _fields_ = [("n_blocks", C.c_int32), ("connectivity", C.c_int32), ("min_area", C.c_int32)]

    def __init__(self, n_blocks=4, connectivity=1, min_area=4):
        super().__init__(n_blocks, connectivity, min_area)


class TRACKER_CFG(C.Structure):
    """trb_tracker_config == TrackerConfig (tracking.hpp:21-34)."""
    _fields_ = [("k_clusters", C.c_int32), ("max_iters", C.c_int32), ("eps", C.c_double),
                ("kmeans_iters", C.c_int32), ("_pad", C.c_int32), ("seed", C.c_uint64)]

    def __init__(self, k_clusters=16, max_iters=20, eps=0.5, kmeans_iters=20, seed=0):
        super().__init__(k_clusters, max_iters, eps, kmeans_iters, 0, seed)


class BLOB(C.Structure):
    _fields_ = [("label", C.c_int32), ("area", C.c_int32), ("x_min", C.c_int32), ("y_min", C.c_int32),
                ("x_max", C.c_int32), ("y_max", C.c_int32), ("cx", C.c_double), ("cy", C.c_double)]


class LOGE(C.Structure):
    _fields_ = [("frame", C.c_int32), ("track_id", C.c_int32), ("x", C.c_double), ("y", C.c_double),
                ("w", C.c_int32), ("h", C.c_int32), ("status", C.c_int32), ("_pad", C.c_int32)]


class TRACK(C.Structure):
    _fields_ = [("track_id", C.c_int32), ("w", C.c_int32), ("h", C.c_int32), ("status", C.c_int32),
                ("lost_frames", C.c_int32), ("k", C.c_int32), ("cx", C.c_double), ("cy", C.c_double)]


class STREAMS_OPTS(C.Structure):
    """trb_streams_options: per-stream track and track-log capacities."""
    _fields_ = [("track_cap", C.c_int32), ("_pad", C.c_int32), ("log_cap", C.c_int64)]

    def __init__(self, track_cap=256, log_cap=1 << 16):
        super().__init__(track_cap, 0, log_cap)


class STEP_OUTPUT(C.Structure):
    """trb_step_output: host (pinned) targets of a step's results."""
    _fields_ = [("n_blobs", C.c_void_p), ("blobs", C.c_void_p), ("blob_cap", C.c_int32), ("log_cap", C.c_int32),
                ("n_log", C.c_void_p), ("log", C.c_void_p)]


BLOB_DTYPE = np.dtype([("label", "<i4"), ("area", "<i4"), ("x_min", "<i4"), ("y_min", "<i4"), ("x_max", "<i4"),
                       ("y_max", "<i4"), ("cx", "<f8"), ("cy", "<f8")])
LOG_DTYPE = np.dtype([("frame", "<i4"), ("track_id", "<i4"), ("x", "<f8"), ("y", "<f8"), ("w", "<i4"),
                      ("h", "<i4"), ("status", "<i4"), ("_pad", "<i4")])
assert BLOB_DTYPE.itemsize == C.sizeof(BLOB) == 40
assert LOG_DTYPE.itemsize == C.sizeof(LOGE) == 40


def blobs_to_array(carr, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, BLOB_DTYPE)
    buf = (C.c_char * (n * C.sizeof(BLOB))).from_address(C.addressof(carr))
    return np.frombuffer(bytes(buf), dtype=BLOB_DTYPE).copy()


def log_to_array(carr, n: int) -> np.ndarray:
    if n == 0:
        return np.zeros(0, LOG_DTYPE)
    buf = (C.c_char * (n * C.sizeof(LOGE))).from_address(C.addressof(carr))
    arr = np.frombuffer(bytes(buf), dtype=LOG_DTYPE).copy()
    arr["_pad"] = 0
    return arr

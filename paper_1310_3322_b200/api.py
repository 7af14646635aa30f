"""Python mirror of the reference's hot-path API over the C ABI (include/trb.h).

Names, argument meaning and error behaviour follow the reference classes so
tests read like the reference's own (motion_test.cpp, segmentation_test.cpp,
tracking_test.cpp):

    MotionDetector(cfg, w, h).push(gray)      motion.hpp:149-212
    label_blocked(mask, w, h, cfg)            segmentation.hpp:198-264
    label_sequential(mask, w, h, cfg)         segmentation.hpp:183-191
    Tracker(cfg).process(frame, w, h, c, blobs)  tracking.hpp:170-241
    meanshift_step / histogram / quantize_colors

Every call runs the sm_100a kernels in ``libtrb.so``; there is no CPU
fallback — a missing library or device raises.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading
from typing import List, Optional, Sequence

import numpy as np

from .abi import (BLOB, BLOB_DTYPE, LOG_DTYPE, LOGE, MOTION_CFG, SEG_CFG, STEP_OUTPUT, STREAMS_OPTS, TRACK,
                  TRACKER_CFG, blobs_to_array, log_to_array)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# TRB_LIB selects another in-tree build of the library (A/B experiments)
LIB_PATH = os.environ.get("TRB_LIB") or os.path.join(PKG_DIR, "libtrb.so")
CSRC = os.path.join(PKG_DIR, "csrc")

MotionConfig = MOTION_CFG
SegmentationConfig = SEG_CFG
TrackerConfig = TRACKER_CFG

MEAN, MODE = 0, 1
FOUR, EIGHT = 0, 1
ACTIVE, LOST = 0, 1
MORPH_NONE, MORPH_ERODE, MORPH_DILATE, MORPH_OPEN, MORPH_CLOSE = range(5)


class TeamrecError(RuntimeError):
    """teamrec::Error (error.hpp:9-12)"""


class InvalidArgument(TeamrecError):
    pass


class ConfigError(TeamrecError):
    pass


class IoError(TeamrecError):
    pass


class CudaError(TeamrecError):
    pass


class CapacityError(TeamrecError):
    pass


_ERRORS = {1: InvalidArgument, 2: ConfigError, 3: IoError, 4: CudaError, 5: CudaError, 6: CapacityError}

_lib = None
_lock = threading.Lock()


def build(force: bool = False) -> str:
    """Compile libtrb.so in-tree for sm_100a (nvcc cross-compiles without a GPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC, "-j8"], check=True)
    return LIB_PATH


def lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                build()
            L = C.CDLL(LIB_PATH)
            _declare(L)
            _lib = L
    return _lib


def _declare(L):
    vp, i32, i64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_double
    L.trb_last_error.restype = C.c_char_p
    L.trb_version.restype = C.c_char_p
    sig = {
        "trb_device_count": [C.POINTER(C.c_int)],
        "trb_motion_config_validate": [C.POINTER(MOTION_CFG)],
        "trb_seg_config_validate": [C.POINTER(SEG_CFG)],
        "trb_tracker_config_validate": [C.POINTER(TRACKER_CFG)],
        "trb_motion_create": [C.POINTER(MOTION_CFG), i32, i32, i32, C.POINTER(vp)],
        "trb_motion_destroy": [vp],
        "trb_motion_push": [vp, vp, i32, i32, i32, i64, vp, C.POINTER(C.c_int)],
        "trb_motion_background": [vp, vp],
        "trb_motion_frames_seen": [vp, C.POINTER(C.c_int)],
        "trb_label": [vp, i32, i32, C.POINTER(SEG_CFG), i32, vp, vp, i32, C.POINTER(C.c_int), vp, i64],
        "trb_tracker_create": [C.POINTER(TRACKER_CFG), i32, C.POINTER(vp)],
        "trb_tracker_destroy": [vp],
        "trb_tracker_process": [vp, vp, i32, i32, i32, vp, i32],
        "trb_tracker_num_tracks": [vp, C.POINTER(C.c_int)],
        "trb_tracker_tracks": [vp, vp, i32],
        "trb_tracker_track_model": [vp, i32, vp, vp],
        "trb_tracker_log_size": [vp, C.POINTER(C.c_int64)],
        "trb_tracker_log": [vp, vp, i64],
        "trb_tracker_frames_processed": [vp, C.POINTER(C.c_int)],
        "trb_streams_create": [i32, i32, i32, i32, C.POINTER(MOTION_CFG), C.POINTER(SEG_CFG),
                               C.POINTER(TRACKER_CFG), i32, C.POINTER(vp)],
        "trb_streams_create_ex": [i32, i32, i32, i32, C.POINTER(MOTION_CFG), C.POINTER(SEG_CFG),
                                  C.POINTER(TRACKER_CFG), C.POINTER(STREAMS_OPTS), i32, C.POINTER(vp)],
        "trb_streams_step_host_async_out": [vp, vp, C.POINTER(STEP_OUTPUT), vp],
        "trb_streams_drain_log": [vp, i32, vp, i64, C.POINTER(C.c_int64)],
        "trb_streams_destroy": [vp],
        "trb_streams_step_device": [vp, vp, vp],
        "trb_streams_step_host": [vp, vp, vp, vp],
        "trb_streams_step_host_async": [vp, vp, vp, vp],
        "trb_warp_frame": [vp, i32, i32, i32, vp, i32, vp],
        "trb_decode_pnm": [vp, i64, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), vp, i64],
        "trb_load_pnm": [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int), vp, i64],
        "trb_load_frame_sequence": [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                    C.POINTER(C.c_int), vp, vp, i64],
        "trb_format_track_log": [vp, i64, vp, i64, C.POINTER(C.c_int64)],
        "trb_parse_track_log": [C.c_char_p, i64, C.c_char_p, vp, i64, C.POINTER(C.c_int64)],
        "trb_save_track_log": [C.c_char_p, vp, i64],
        "trb_load_track_log": [C.c_char_p, vp, i64, C.POINTER(C.c_int64)],
        "trb_streams_step_device_warp": [vp, vp, vp, vp],
        "trb_extract_blob_features": [vp, i32, i32, vp, i32, i32, i32, vp, i32, i32, vp, vp],
        "trb_streams_blob_features": [vp, i32, vp, vp, vp, i32, C.POINTER(C.c_int)],
        "trb_morph_device": [vp, vp, i32, i32, i32, i32, vp],
        "trb_streams_synchronize": [vp],
        "trb_streams_join": [vp, vp],
        "trb_streams_frames_seen": [vp, C.POINTER(C.c_int)],
        "trb_streams_has_output": [vp, C.POINTER(C.c_int)],
        "trb_streams_download_mask": [vp, i32, vp],
        "trb_streams_download_labels": [vp, i32, vp],
        "trb_streams_download_blobs": [vp, i32, vp, i32, C.POINTER(C.c_int)],
        "trb_streams_log_size": [vp, i32, C.POINTER(C.c_int64)],
        "trb_streams_download_log": [vp, i32, vp, i64],
        "trb_streams_num_tracks": [vp, i32, C.POINTER(C.c_int)],
        "trb_streams_last_step_launches": [vp, C.POINTER(C.c_int)],
        "trb_streams_device_planes": [vp, i32, vp, vp],
        "trb_streams_profile": [vp, i32],
        "trb_streams_profile_read": [vp, vp, C.POINTER(C.c_int)],
        "trb_synth_raster": [vp, i32, i32, i32, C.c_uint8, vp, vp, i32, vp],
        "trb_synth_raster_frames": [vp, i64, i32, i32, i32, i32, C.c_uint8, vp, vp, i32, vp],
        "trb_meanshift_step": [vp, i32, i32, i32, C.POINTER(dbl), C.POINTER(dbl), i32, i32, vp, vp, i32, i32, dbl,
                               C.POINTER(C.c_int), i32],
        "trb_histogram": [vp, i32, i32, i32, dbl, dbl, i32, i32, vp, i32, i32, vp, i32],
        "trb_quantize_colors": [vp, i64, i32, i32, C.c_uint64, vp, i32],
        "trb_selftest_hypot": [vp, vp, i64, vp, i32],
        "trb_debug_stats": [vp, i32],
        "trb_debug_progress": [i32, vp],
        "trb_debug_itlog": [i32, vp, i64, C.POINTER(C.c_int64)],
        "trb_debug_phases": [vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = C.c_int
    for name in ("trb_default_motion_config", "trb_default_seg_config", "trb_default_tracker_config",
                 "trb_default_streams_options"):
        getattr(L, name).restype = None


def _check(rc: int) -> None:
    if rc != 0:
        msg = lib().trb_last_error().decode()
        raise _ERRORS.get(rc, TeamrecError)(msg)


def _ptr(a: np.ndarray):
    return C.c_void_p(a.ctypes.data)


def device_count() -> int:
    n = C.c_int(0)
    _check(lib().trb_device_count(C.byref(n)))
    return n.value


# ---------------------------------------------------------------- motion
class MotionDetector:
    """MotionDetector (motion.hpp:149-212) on the GPU."""

    def __init__(self, cfg: Optional[MOTION_CFG] = None, width: int = 0, height: int = 0, device: int = 0):
        self.cfg = cfg if cfg is not None else MOTION_CFG()
        self.width, self.height = width, height
        h = C.c_void_p()
        _check(lib().trb_motion_create(C.byref(self.cfg), width, height, device, C.byref(h)))
        self._h = h

    def push(self, gray: np.ndarray, channels: int = 1, width: Optional[int] = None, height: Optional[int] = None,
             index: int = 0) -> Optional[np.ndarray]:
        g = np.ascontiguousarray(gray, dtype=np.uint8).reshape(-1)
        w = self.width if width is None else width
        h = self.height if height is None else height
        out = np.empty(self.width * self.height, np.uint8)
        has = C.c_int(0)
        _check(lib().trb_motion_push(self._h, _ptr(g), w, h, channels, index, _ptr(out), C.byref(has)))
        return out if has.value else None

    def background(self) -> np.ndarray:
        out = np.empty(self.width * self.height, np.uint8)
        _check(lib().trb_motion_background(self._h, _ptr(out)))
        return out

    @property
    def frames_seen(self) -> int:
        n = C.c_int(0)
        _check(lib().trb_motion_frames_seen(self._h, C.byref(n)))
        return n.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.trb_motion_destroy(self._h)
            self._h = None


# ------------------------------------------------------------- labelling
class Labeling:
    """Labeling (segmentation.hpp:47-54): labels int32[h*w], blobs (structured
    array with BLOB_DTYPE fields), optional per-blob pixel lists."""

    def __init__(self, width, height, labels, blobs, pixels=None):
        self.width, self.height, self.labels, self.blobs = width, height, labels, blobs
        self._pixels = pixels

    def blob_pixels(self, k: int) -> np.ndarray:
        if self._pixels is None:
            raise InvalidArgument("pixel lists were not requested")
        off = np.concatenate([[0], np.cumsum(self.blobs["area"].astype(np.int64))])
        return self._pixels[off[k]:off[k + 1]]

    def label_at(self, x: int, y: int) -> int:
        return int(self.labels[y * self.width + x])


def label_blocked(mask: np.ndarray, width: int, height: int, cfg: Optional[SEG_CFG] = None, device: int = 0,
                  want_pixels: bool = False) -> Labeling:
    cfg = cfg if cfg is not None else SEG_CFG()
    m = np.ascontiguousarray(mask, dtype=np.uint8).reshape(-1)
    if m.size != width * height:
        raise InvalidArgument("mask data length does not match width*height")
    labels = np.empty(width * height, np.int32)
    cap = max(16, width * height // 2 + 1)
    blobs = (BLOB * cap)()
    n = C.c_int(0)
    pixels = None
    pp, pcap = None, 0
    if want_pixels:
        pixels = np.empty(int(np.count_nonzero(m)) + 1, np.int64)
        pp, pcap = _ptr(pixels), pixels.size
    _check(lib().trb_label(_ptr(m), width, height, C.byref(cfg), device, _ptr(labels), blobs, cap, C.byref(n), pp,
                           pcap))
    arr = blobs_to_array(blobs, n.value)
    if want_pixels:
        pixels = pixels[:int(arr["area"].sum())]
    return Labeling(width, height, labels, arr, pixels)


def label_sequential(mask: np.ndarray, width: int, height: int, cfg: Optional[SEG_CFG] = None, device: int = 0,
                     want_pixels: bool = False) -> Labeling:
    """label_sequential (segmentation.hpp:183-191): same output, no grid check."""
    cfg = cfg if cfg is not None else SEG_CFG()
    _check(lib().trb_seg_config_validate(C.byref(cfg)))
    c = SEG_CFG(1, cfg.connectivity, cfg.min_area)
    return label_blocked(mask, width, height, c, device, want_pixels)


# --------------------------------------------------------------- tracker
class Tracker:
    """Tracker (tracking.hpp:170-241) with all state on the GPU."""

    def __init__(self, cfg: Optional[TRACKER_CFG] = None, device: int = 0):
        self.cfg = cfg if cfg is not None else TRACKER_CFG()
        h = C.c_void_p()
        _check(lib().trb_tracker_create(C.byref(self.cfg), device, C.byref(h)))
        self._h = h

    def process(self, frame: np.ndarray, width: int, height: int, channels: int, blobs) -> None:
        f = np.ascontiguousarray(frame, dtype=np.uint8).reshape(-1)
        b = np.ascontiguousarray(blobs if isinstance(blobs, np.ndarray) else np.array(blobs, dtype=BLOB_DTYPE),
                                 dtype=BLOB_DTYPE)
        _check(lib().trb_tracker_process(self._h, _ptr(f), width, height, channels,
                                         _ptr(b) if b.size else None, int(b.size)))

    def tracks(self) -> List[TRACK]:
        n = C.c_int(0)
        _check(lib().trb_tracker_num_tracks(self._h, C.byref(n)))
        arr = (TRACK * max(1, n.value))()
        _check(lib().trb_tracker_tracks(self._h, arr, n.value))
        return [arr[i] for i in range(n.value)]

    def track_model(self, i: int):
        k = self.cfg.k_clusters
        c = np.empty(3 * k)
        q = np.empty(k)
        _check(lib().trb_tracker_track_model(self._h, i, _ptr(c), _ptr(q)))
        return c.reshape(k, 3), q

    def log(self) -> np.ndarray:
        n = C.c_int64(0)
        _check(lib().trb_tracker_log_size(self._h, C.byref(n)))
        arr = (LOGE * max(1, n.value))()
        _check(lib().trb_tracker_log(self._h, arr, n.value))
        return log_to_array(arr, n.value)

    @property
    def frames_processed(self) -> int:
        n = C.c_int(0)
        _check(lib().trb_tracker_frames_processed(self._h, C.byref(n)))
        return n.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.trb_tracker_destroy(self._h)
            self._h = None


def meanshift_step(frame: np.ndarray, width: int, height: int, channels: int, cx: float, cy: float, w: int, h: int,
                   centers: np.ndarray, target: np.ndarray, max_iters: int = 20, eps: float = 0.5,
                   status: int = ACTIVE, device: int = 0):
    """meanshift_step (tracking.hpp:125-157) -> (cx, cy, status)."""
    f = np.ascontiguousarray(frame, dtype=np.uint8).reshape(-1)
    c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1)
    q = np.ascontiguousarray(target, dtype=np.float64).reshape(-1)
    x, y, st = C.c_double(cx), C.c_double(cy), C.c_int(status)
    _check(lib().trb_meanshift_step(_ptr(f), width, height, channels, C.byref(x), C.byref(y), w, h, _ptr(c), _ptr(q),
                                    q.size, max_iters, eps, C.byref(st), device))
    return x.value, y.value, st.value


# ------------------------------------------------------------------ I/O
def decode_pnm(data: bytes, source_name: str = "<memory>"):
    """decode_pnm (frame.hpp:152-175) -> (pixels uint8[w*h*ch], w, h, ch)."""
    buf = np.frombuffer(bytes(data), np.uint8) if len(data) else np.zeros(1, np.uint8)
    w, h, c = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib().trb_decode_pnm(_ptr(buf), len(data), source_name.encode(), C.byref(w), C.byref(h), C.byref(c),
                                None, 0))
    out = np.empty(w.value * h.value * c.value, np.uint8)
    _check(lib().trb_decode_pnm(_ptr(buf), len(data), source_name.encode(), C.byref(w), C.byref(h), C.byref(c),
                                _ptr(out), out.size))
    return out, w.value, h.value, c.value


def load_pnm(path: str):
    """load_pnm (frame.hpp:177-182) -> (pixels, w, h, ch)."""
    w, h, c = C.c_int(0), C.c_int(0), C.c_int(0)
    _check(lib().trb_load_pnm(str(path).encode(), C.byref(w), C.byref(h), C.byref(c), None, 0))
    out = np.empty(w.value * h.value * c.value, np.uint8)
    _check(lib().trb_load_pnm(str(path).encode(), C.byref(w), C.byref(h), C.byref(c), _ptr(out), out.size))
    return out, w.value, h.value, c.value


def load_frame_sequence(directory: str):
    """load_frame_sequence (frame.hpp:198-225) -> (frames [n, w*h*ch], indices, w, h, ch)."""
    n, w, h, c = C.c_int(0), C.c_int(0), C.c_int(0), C.c_int(0)
    d = str(directory).encode()
    _check(lib().trb_load_frame_sequence(d, C.byref(n), C.byref(w), C.byref(h), C.byref(c), None, None, 0))
    fb = w.value * h.value * c.value
    out = np.empty((n.value, fb), np.uint8)
    idx = np.empty(max(1, n.value), np.int64)
    _check(lib().trb_load_frame_sequence(d, C.byref(n), C.byref(w), C.byref(h), C.byref(c), _ptr(idx), _ptr(out),
                                         out.size))
    return out, idx[:n.value], w.value, h.value, c.value


def format_track_log(log) -> str:
    """format_track_log (tracking.hpp:247-256)."""
    a = np.ascontiguousarray(log, dtype=LOG_DTYPE)
    n = C.c_int64(0)
    _check(lib().trb_format_track_log(_ptr(a) if len(a) else None, len(a), None, 0, C.byref(n)))
    buf = C.create_string_buffer(n.value + 1)
    _check(lib().trb_format_track_log(_ptr(a) if len(a) else None, len(a), buf, n.value + 1, C.byref(n)))
    return buf.value.decode()


def parse_track_log(text: str, source: str = "<memory>") -> np.ndarray:
    """parse_track_log (tracking.hpp:258-277) -> structured log array."""
    t = text.encode()
    n = C.c_int64(0)
    _check(lib().trb_parse_track_log(t, len(t), source.encode(), None, 0, C.byref(n)))
    out = np.zeros(n.value, LOG_DTYPE)
    _check(lib().trb_parse_track_log(t, len(t), source.encode(), _ptr(out) if n.value else None, n.value,
                                     C.byref(n)))
    return out


def save_track_log(log, path: str) -> None:
    a = np.ascontiguousarray(log, dtype=LOG_DTYPE)
    _check(lib().trb_save_track_log(str(path).encode(), _ptr(a) if len(a) else None, len(a)))


def load_track_log(path: str) -> np.ndarray:
    n = C.c_int64(0)
    _check(lib().trb_load_track_log(str(path).encode(), None, 0, C.byref(n)))
    out = np.zeros(n.value, LOG_DTYPE)
    _check(lib().trb_load_track_log(str(path).encode(), _ptr(out) if n.value else None, n.value, C.byref(n)))
    return out


def warp_frame(frame: np.ndarray, width: int, height: int, channels: int, homography, device: int = 0) -> np.ndarray:
    """warp_frame (motion.hpp:81-119): inverse-mapped bilinear resampling by
    the 3x3 homography (samples off the source plane read 0)."""
    f = np.ascontiguousarray(frame, dtype=np.uint8).reshape(-1)
    hm = np.ascontiguousarray(homography, dtype=np.float64).reshape(9)
    out = np.empty(width * height * channels, np.uint8)
    _check(lib().trb_warp_frame(_ptr(f), width, height, channels, _ptr(hm), device, _ptr(out)))
    return out


def extract_blob_features(labels: np.ndarray, width: int, height: int, frame: np.ndarray, frame_width: int,
                          frame_height: int, channels: int, blobs, device: int = 0):
    """extract_blob_features (segmentation.hpp:268-291) -> (mean_intensity,
    aspect) arrays, one entry per blob record."""
    lab = np.ascontiguousarray(labels, dtype=np.int32).reshape(-1)
    f = np.ascontiguousarray(frame, dtype=np.uint8).reshape(-1)
    b = np.ascontiguousarray(blobs)
    n = len(b)
    mean, aspect = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    _check(lib().trb_extract_blob_features(_ptr(lab), width, height, _ptr(f), frame_width, frame_height, channels,
                                           _ptr(b) if n else None, n, device, _ptr(mean), _ptr(aspect)))
    return mean[:n], aspect[:n]


def histogram(frame: np.ndarray, width: int, height: int, channels: int, cx: float, cy: float, w: int, h: int,
              centers: np.ndarray, epanechnikov: bool = True, device: int = 0) -> np.ndarray:
    """histogram (tracking.hpp:106-112)."""
    f = np.ascontiguousarray(frame, dtype=np.uint8).reshape(-1)
    c = np.ascontiguousarray(centers, dtype=np.float64).reshape(-1)
    k = c.size // 3
    out = np.empty(k)
    _check(lib().trb_histogram(_ptr(f), width, height, channels, cx, cy, w, h, _ptr(c), k, int(epanechnikov),
                               _ptr(out), device))
    return out


def quantize_colors(pixels: np.ndarray, k: int, iters: int, seed: int, device: int = 0) -> np.ndarray:
    """quantize_colors (quantize.hpp:43-118) -> centres (k, 3)."""
    p = np.ascontiguousarray(pixels, dtype=np.float64).reshape(-1, 3)
    out = np.empty(3 * k)
    _check(lib().trb_quantize_colors(_ptr(p), p.shape[0], k, iters, seed, _ptr(out), device))
    return out.reshape(k, 3)


# --------------------------------------------------------------- streams
class StepOutput:
    """Pinned host targets for one step's results (trb_step_output): per
    stream the blob count, the first `blob_cap` blobs and the log entries
    the frame appended (first `log_cap`).  Read after Streams.synchronize()."""

    def __init__(self, n_streams: int, blob_cap: int = 64, log_cap: int = 32):
        import torch  # pinned host memory (cudaMallocHost through torch's caching host allocator)
        self.n, self.blob_cap, self.log_cap = n_streams, blob_cap, log_cap
        pin = lambda nbytes: torch.empty(max(16, nbytes), dtype=torch.uint8).pin_memory()
        self._bufs = [pin(4 * n_streams), pin(4 * n_streams), pin(BLOB_DTYPE.itemsize * n_streams * blob_cap),
                      pin(LOG_DTYPE.itemsize * n_streams * log_cap)]
        b = self._bufs
        self.n_blobs = b[0].numpy()[:4 * n_streams].view(np.int32)
        self.n_log = b[1].numpy()[:4 * n_streams].view(np.int32)
        self.blobs = b[2].numpy()[:BLOB_DTYPE.itemsize * n_streams * blob_cap].view(BLOB_DTYPE).reshape(
            n_streams, blob_cap)
        self.log = b[3].numpy()[:LOG_DTYPE.itemsize * n_streams * log_cap].view(LOG_DTYPE).reshape(n_streams, log_cap)
        self.c = STEP_OUTPUT(b[0].data_ptr(), b[2].data_ptr() if blob_cap else None, blob_cap, log_cap,
                             b[1].data_ptr(), b[3].data_ptr() if log_cap else None)

    @property
    def nbytes(self) -> int:
        """Bytes the device writes back per step."""
        return 8 * self.n + (BLOB_DTYPE.itemsize * self.blob_cap + LOG_DTYPE.itemsize * self.log_cap) * self.n

    def stream_blobs(self, s: int) -> np.ndarray:
        return self.blobs[s, :min(int(self.n_blobs[s]), self.blob_cap)].copy()

    def stream_log(self, s: int) -> np.ndarray:
        return self.log[s, :min(int(self.n_log[s]), self.log_cap)].copy()


class Streams:
    """The batched device-resident front end (run_vision, harness.hpp:412-450)
    for n independent streams of one geometry.  track_cap / log_cap bound the
    live tracks and the undrained track-log entries per stream
    (trb_streams_options); exceeding either fails the step (CapacityError)."""

    def __init__(self, n_streams: int, width: int, height: int, channels: int = 1,
                 motion: Optional[MOTION_CFG] = None, seg: Optional[SEG_CFG] = None,
                 tracker: Optional[TRACKER_CFG] = TRACKER_CFG(), device: int = 0, track_cap: int = 256,
                 log_cap: int = 1 << 16):
        self.n, self.width, self.height, self.channels = n_streams, width, height, channels
        self.motion = motion if motion is not None else MOTION_CFG()
        self.seg = seg if seg is not None else SEG_CFG()
        self.tracker = tracker
        self.opts = STREAMS_OPTS(track_cap, log_cap)
        h = C.c_void_p()
        _check(lib().trb_streams_create_ex(n_streams, width, height, channels, C.byref(self.motion),
                                           C.byref(self.seg), C.byref(tracker) if tracker is not None else None,
                                           C.byref(self.opts), device, C.byref(h)))
        self._h = h
        self._ptrs = (C.c_void_p * n_streams)()

    def _frame_count(self, frames) -> None:
        if len(frames) != self.n:
            raise InvalidArgument(f"expected {self.n} frames (one per stream), got {len(frames)}")

    def _host_frames(self, frames, ptrs) -> None:
        """Host frames: C-contiguous uint8 arrays of width*height*channels."""
        self._frame_count(frames)
        need = self.width * self.height * self.channels
        for i, f in enumerate(frames):
            if not isinstance(f, np.ndarray) or f.dtype != np.uint8 or not f.flags["C_CONTIGUOUS"] or f.size != need:
                raise InvalidArgument(f"frame {i}: expected a C-contiguous uint8 array of {need} bytes")
            ptrs[i] = f.ctypes.data

    def step_device(self, frame_ptrs: Sequence[int], cuda_stream: int = 0) -> None:
        self._frame_count(frame_ptrs)
        for i, p in enumerate(frame_ptrs):
            self._ptrs[i] = p
        _check(lib().trb_streams_step_device(self._h, self._ptrs, C.c_void_p(cuda_stream)))

    def step_device_warp(self, frame_ptrs: Sequence[int], homographies, cuda_stream: int = 0) -> None:
        """MotionConfig(warp=1): warp every stream's frame by its homography
        (n_streams x 3 x 3) before it enters the window (stream_detect)."""
        self._frame_count(frame_ptrs)
        for i, p in enumerate(frame_ptrs):
            self._ptrs[i] = p
        hm = np.ascontiguousarray(homographies, dtype=np.float64).reshape(-1)
        if hm.size != 9 * self.n:
            raise InvalidArgument(f"expected {self.n} homographies (3x3 each)")
        _check(lib().trb_streams_step_device_warp(self._h, self._ptrs, _ptr(hm), C.c_void_p(cuda_stream)))

    def _result(self, result):
        if result is None:
            return None
        if result.dtype != np.int32 or result.size < self.n or not result.flags["C_CONTIGUOUS"]:
            raise InvalidArgument(f"result: expected a contiguous int32 array of {self.n} entries")
        return _ptr(result)

    def step_host(self, frames: Sequence[np.ndarray], result: Optional[np.ndarray] = None,
                  cuda_stream: int = 0) -> None:
        self._host_frames(frames, self._ptrs)
        _check(lib().trb_streams_step_host(self._h, self._ptrs, self._result(result), C.c_void_p(cuda_stream)))

    def step_host_async(self, frames: Sequence[np.ndarray], result=None, cuda_stream: int = 0) -> None:
        """Pipelined step_host: queued work only; `frames` and `result` must
        stay alive (and unmodified) until synchronize().  `result` is an int32
        array (blob counts) or a StepOutput (blob tables + the frame's log
        entries)."""
        ptrs = (C.c_void_p * self.n)()
        self._host_frames(frames, ptrs)
        if isinstance(result, StepOutput):
            if result.n != self.n:
                raise InvalidArgument("StepOutput was made for another stream count")
            _check(lib().trb_streams_step_host_async_out(self._h, ptrs, C.byref(result.c), C.c_void_p(cuda_stream)))
            return
        _check(lib().trb_streams_step_host_async(self._h, ptrs, self._result(result), C.c_void_p(cuda_stream)))

    def num_tracks(self, s: int) -> int:
        """Live tracks of stream s (Tracker::tracks().size())."""
        n = C.c_int(0)
        _check(lib().trb_streams_num_tracks(self._h, s, C.byref(n)))
        return n.value

    def drain_log(self, s: int) -> np.ndarray:
        """The track-log entries of stream s not drained yet (oldest first);
        they are released from the device ring."""
        n = C.c_int64(0)
        _check(lib().trb_streams_log_size(self._h, s, C.byref(n)))
        arr = (LOGE * max(1, n.value))()
        got = C.c_int64(0)
        _check(lib().trb_streams_drain_log(self._h, s, arr, n.value, C.byref(got)))
        return log_to_array(arr, got.value)

    def synchronize(self) -> None:
        _check(lib().trb_streams_synchronize(self._h))

    def join(self, cuda_stream: int = 0) -> None:
        """Make cuda_stream wait (on the device) for every step issued so far
        (a step's tracking overlaps the next step's motion + CCL on an
        internal stream; trb_streams_join)."""
        _check(lib().trb_streams_join(self._h, C.c_void_p(cuda_stream)))

    @property
    def has_output(self) -> bool:
        v = C.c_int(0)
        _check(lib().trb_streams_has_output(self._h, C.byref(v)))
        return bool(v.value)

    @property
    def last_launches(self) -> int:
        v = C.c_int(0)
        _check(lib().trb_streams_last_step_launches(self._h, C.byref(v)))
        return v.value

    def mask(self, s: int) -> np.ndarray:
        out = np.empty(self.width * self.height, np.uint8)
        _check(lib().trb_streams_download_mask(self._h, s, _ptr(out)))
        return out

    def labels(self, s: int) -> np.ndarray:
        out = np.empty(self.width * self.height, np.int32)
        _check(lib().trb_streams_download_labels(self._h, s, _ptr(out)))
        return out

    def blobs(self, s: int) -> np.ndarray:
        n = C.c_int(0)
        _check(lib().trb_streams_download_blobs(self._h, s, None, 0, C.byref(n)))
        arr = (BLOB * max(1, n.value))()
        _check(lib().trb_streams_download_blobs(self._h, s, arr, n.value, C.byref(n)))
        return blobs_to_array(arr, n.value)

    def log(self, s: int) -> np.ndarray:
        n = C.c_int64(0)
        _check(lib().trb_streams_log_size(self._h, s, C.byref(n)))
        arr = (LOGE * max(1, n.value))()
        _check(lib().trb_streams_download_log(self._h, s, arr, n.value))
        return log_to_array(arr, n.value)

    def profile(self, enable: bool) -> None:
        _check(lib().trb_streams_profile(self._h, int(enable)))

    def profile_read(self):
        """-> (ms per stage [motion, ccl, meanshift, gate+spawn] summed, steps)"""
        ms = np.zeros(4)
        n = C.c_int(0)
        _check(lib().trb_streams_profile_read(self._h, _ptr(ms), C.byref(n)))
        return ms, n.value

    def blob_features(self, s: int, frame_device_ptr: int):
        """extract_blob_features of stream s's last step (frame_device_ptr:
        that step's frame in HBM) -> (mean_intensity, aspect)."""
        cap = self.width * self.height // 2 + 2
        mean, aspect = np.zeros(cap), np.zeros(cap)
        n = C.c_int(0)
        _check(lib().trb_streams_blob_features(self._h, s, C.c_void_p(frame_device_ptr), _ptr(mean), _ptr(aspect),
                                               cap, C.byref(n)))
        return mean[:n.value], aspect[:n.value]

    def device_planes(self, s: int):
        m, l_ = C.c_void_p(), C.c_void_p()
        _check(lib().trb_streams_device_planes(self._h, s, C.byref(m), C.byref(l_)))
        return m.value, l_.value

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.trb_streams_destroy(self._h)
            self._h = None


def synth_raster(out_device_ptr: int, width: int, height: int, channels: int, background: int, rects, colors,
                 cuda_stream: int = 0) -> None:
    """Device raster of one synthetic frame (synth.hpp:295-328)."""
    r = np.ascontiguousarray(np.asarray(rects, dtype=np.int32).reshape(-1))
    c = np.ascontiguousarray(np.asarray(colors, dtype=np.uint8).reshape(-1))
    _check(lib().trb_synth_raster(C.c_void_p(out_device_ptr), width, height, channels, background, _ptr(r), _ptr(c),
                                  r.size // 4, C.c_void_p(cuda_stream)))


STAT_NAMES = ("osum_calls", "osum_sums", "osum_fallback_sums", "osum_breakpoints", "osum_elements",
              "meanshift_iters", "spawns", "lloyd_iters", "empty_cluster_passes", "tracks_advanced",
              "", "meanshift_window_px", "fast_warps", "", "general_warps", "",
              "bad_scan_merge", "bad_phaseB_merge", "bad_bp_overflow", "bad_cross_cta", "bad_fold_carry",
              "bad_fold_merge", "bad_verify_start", "bad_verify_end", "rec_fixed_lanes", "rec_selected_lanes",
              "rec_heads", "", "max_bp_cta", "max_bp")


def debug_stats(reset: bool = False) -> dict:
    out = np.zeros(32, np.uint64)
    _check(lib().trb_debug_stats(_ptr(out), int(reset)))
    return {k: int(v) for k, v in zip(STAT_NAMES, out) if k and int(v)}


def debug_progress(n_ctas: int = 4096):
    """Host-mapped progress records of the tracker CTAs ([n, 4] int view)."""
    p = C.POINTER(C.c_int)()
    _check(lib().trb_debug_progress(n_ctas, C.byref(p)))
    return np.ctypeslib.as_array(p, shape=(n_ctas, 4))


def synth_raster_frames(out_device_ptr: int, frame_stride: int, width: int, height: int, channels: int,
                        background: int, rects_per_frame, colors, cuda_stream: int = 0) -> None:
    """Device raster of many frames of one clip in a single launch."""
    r = np.ascontiguousarray(np.asarray(rects_per_frame, dtype=np.int32))
    n_frames = r.shape[0]
    c = np.ascontiguousarray(np.asarray(colors, dtype=np.uint8).reshape(-1))
    _check(lib().trb_synth_raster_frames(C.c_void_p(out_device_ptr), frame_stride, n_frames, width, height, channels,
                                         background, _ptr(r), _ptr(c), r.shape[1], C.c_void_p(cuda_stream)))


def debug_itlog(enable=None):
    """enable=True/False toggles; returns the (pixels, cycles) pairs so far."""
    out = np.zeros((1 << 16, 2), np.int64)
    n = C.c_int64(0)
    _check(lib().trb_debug_itlog(-1 if enable is None else int(enable), _ptr(out), 1 << 16, C.byref(n)))
    return out[:n.value]


def debug_phases() -> np.ndarray:
    """Per-phase SM cycles of the logged mean-shift iterations, [4, 32] by
    window-size bucket (<5k, <50k, <150k, larger); [:, 0] = iterations."""
    out = np.zeros(256, np.uint64)
    _check(lib().trb_debug_phases(_ptr(out)))
    return out.reshape(4, 64)


def selftest_hypot(x: np.ndarray, y: np.ndarray, on_device: bool) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.ascontiguousarray(y, dtype=np.float64)
    out = np.empty_like(x)
    _check(lib().trb_selftest_hypot(_ptr(x), _ptr(y), x.size, _ptr(out), int(on_device)))
    return out


def morph_device(in_ptr: int, out_ptr: int, width: int, height: int, n_planes: int, op: int,
                 cuda_stream: int = 0) -> None:
    """3x3 morphology on device masks (trb_morph_device); op = TRB_MORPH_*."""
    _check(lib().trb_morph_device(C.c_void_p(in_ptr), C.c_void_p(out_ptr), width, height, n_planes, op,
                                  C.c_void_p(cuda_stream)))

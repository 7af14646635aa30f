"""TEST INFRASTRUCTURE: ctypes bindings for the CPU checkers.

* ``Orc``  — oracle/liborc.so, the plain-C restatement (oracle/trb_oracle.c)
* ``Ref``  — oracle/_ref/libteamrec_ref.so, the unmodified reference headers
             behind a C shim (oracle/ref_driver.cpp)

Both expose the same small surface (motion detector, labelling, tracker,
synth) so tests can run the same case through either and through the CUDA
product (paper_1310_3322_b200).  Only tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline leg import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
ORC_SO = os.path.join(ORACLE_DIR, "liborc.so")
REF_SO = os.path.join(ORACLE_DIR, "_ref", "libteamrec_ref.so")

from paper_1310_3322_b200.abi import (BLOB, BLOB_DTYPE, LOG_DTYPE, LOGE, MOTION_CFG, SEG_CFG, TRACK, TRACKER_CFG, blobs_to_array,  # noqa: E402
                                      log_to_array)


def build_oracle() -> None:
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _u8p(a):
    return a.ctypes.data_as(C.POINTER(C.c_uint8))


def _i32p(a):
    return a.ctypes.data_as(C.POINTER(C.c_int32))


def _f64p(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


_orc = None
_ref = None


def orc_lib():
    global _orc
    if _orc is None:
        if not os.path.exists(ORC_SO):
            build_oracle()
        L = C.CDLL(ORC_SO)
        vp = C.c_void_p
        L.orc_motion_create.restype = vp
        L.orc_motion_create.argtypes = [C.POINTER(MOTION_CFG), C.c_int, C.c_int]
        L.orc_motion_destroy.argtypes = [vp]
        L.orc_motion_push.argtypes = [vp, C.c_void_p, C.c_void_p]
        L.orc_motion_background.argtypes = [vp, C.c_void_p]
        L.orc_window_background.restype = C.c_uint8
        L.orc_window_background.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int]
        L.orc_grayscale.argtypes = [C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_morph.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p]
        L.orc_label.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_void_p]
        L.orc_quantize_colors.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        L.orc_quantizer_assign.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_double, C.c_double]
        L.orc_histogram.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.orc_mix_seed.restype = C.c_uint64
        L.orc_mix_seed.argtypes = [C.c_uint64, C.c_uint64]
        L.orc_tracker_create.restype = vp
        L.orc_tracker_create.argtypes = [C.POINTER(TRACKER_CFG)]
        L.orc_tracker_destroy.argtypes = [vp]
        L.orc_tracker_process.argtypes = [vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.orc_tracker_num_tracks.argtypes = [vp]
        L.orc_tracker_tracks.argtypes = [vp, C.c_void_p]
        L.orc_tracker_track_model.argtypes = [vp, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_tracker_log_size.restype = C.c_int64
        L.orc_tracker_log_size.argtypes = [vp]
        L.orc_tracker_log.argtypes = [vp, C.c_void_p]
        L.orc_meanshift_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.orc_synth_create.restype = vp
        L.orc_synth_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint8, C.c_int, C.c_void_p, C.c_void_p,
                                       C.c_uint64]
        L.orc_synth_destroy.argtypes = [vp]
        L.orc_synth_next.argtypes = [vp, C.c_void_p, C.c_void_p]
        L.orc_warp_frame.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_blob_features.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                        C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.orc_plane_hash.restype = C.c_uint64
        L.orc_plane_hash.argtypes = [C.c_void_p, C.c_int64]
        L.orc_libm_hypot_n.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.orc_libm_hypot.restype = C.c_double
        L.orc_libm_hypot.argtypes = [C.c_double, C.c_double]
        _orc = L
    return _orc


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref_lib():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        vp = C.c_void_p
        L.ref_last_error.restype = C.c_char_p
        L.ref_motion_create.restype = vp
        L.ref_motion_create.argtypes = [C.POINTER(MOTION_CFG), C.c_int, C.c_int]
        L.ref_motion_destroy.argtypes = [vp]
        L.ref_motion_push.argtypes = [vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int64, C.c_void_p,
                                      C.POINTER(C.c_int)]
        L.ref_motion_background.argtypes = [vp, C.c_void_p]
        L.ref_label.argtypes = [C.c_void_p, C.c_int, C.c_int, C.POINTER(SEG_CFG), C.c_int, C.c_int, C.c_void_p,
                                C.c_void_p, C.c_int, C.POINTER(C.c_int), C.c_void_p]
        L.ref_quantize_colors.argtypes = [C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        L.ref_warp_frame.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_stream_detect.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                        C.POINTER(MOTION_CFG), C.c_void_p, C.POINTER(C.c_int)]
        L.ref_decode_pnm.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int),
                                     C.POINTER(C.c_int), C.c_void_p, C.c_int64]
        L.ref_load_frame_sequence.argtypes = [C.c_char_p, C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int),
                                              C.POINTER(C.c_int), C.c_void_p, C.c_void_p, C.c_int64]
        L.ref_format_track_log.restype = C.c_int64
        L.ref_format_track_log.argtypes = [C.c_void_p, C.c_int64, C.c_char_p, C.c_int64]
        L.ref_parse_track_log.argtypes = [C.c_char_p, C.c_int64, C.c_char_p, C.c_void_p, C.c_int64,
                                          C.POINTER(C.c_int64)]
        L.ref_blob_features.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                        C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_histogram.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_int, C.c_int,
                                    C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        L.ref_meanshift_step.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double),
                                         C.POINTER(C.c_double), C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                         C.c_int, C.c_double, C.POINTER(C.c_int)]
        L.ref_tracker_create.restype = vp
        L.ref_tracker_create.argtypes = [C.POINTER(TRACKER_CFG)]
        L.ref_tracker_destroy.argtypes = [vp]
        L.ref_tracker_process.argtypes = [vp, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int]
        L.ref_tracker_num_tracks.argtypes = [vp]
        L.ref_tracker_tracks.argtypes = [vp, C.c_void_p]
        L.ref_tracker_track_model.argtypes = [vp, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_tracker_log_size.restype = C.c_int64
        L.ref_tracker_log_size.argtypes = [vp]
        L.ref_tracker_log.argtypes = [vp, C.c_void_p]
        L.ref_synth.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint8, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                C.c_uint64, C.c_void_p, C.c_void_p]
        L.ref_run_streams.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                      C.POINTER(MOTION_CFG), C.POINTER(SEG_CFG), C.POINTER(TRACKER_CFG), C.c_void_p,
                                      C.POINTER(C.c_double), C.c_void_p, C.c_void_p]
        L.ref_run_streams_detail.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                             C.POINTER(MOTION_CFG), C.POINTER(SEG_CFG), C.POINTER(TRACKER_CFG),
                                             C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                                             C.c_int64, C.c_void_p]
        _ref = L
    return _ref


def libm_hypot(x: np.ndarray, y: np.ndarray) -> np.ndarray:
    """The live glibc hypot, element by element (C loop)."""
    x = np.ascontiguousarray(x, np.float64)
    y = np.ascontiguousarray(y, np.float64)
    out = np.empty_like(x)
    orc_lib().orc_libm_hypot_n(x.ctypes.data, y.ctypes.data, x.size, out.ctypes.data)
    return out


def plane_hash(a: np.ndarray) -> int:
    """oracle/plane_hash.h digest of an array's bytes."""
    a = np.ascontiguousarray(a)
    return int(orc_lib().orc_plane_hash(a.ctypes.data, a.nbytes))


def ref_run_streams_detail(frames_per_stream, w, h, ch, mcfg, scfg, tcfg, threads, bcap=64, lcap=4096):
    """The unmodified reference per-frame loop (push -> label_blocked ->
    Tracker::process) over each stream's frames ([n_frames, w*h*ch] uint8),
    streams on `threads` host threads.  Per stream: dict(hashes [k,2] of
    mask/labels per steady frame, nblobs [k], blobs [k, bcap], log)."""
    L = ref_lib()
    S = len(frames_per_stream)
    nf = frames_per_stream[0].shape[0]
    ptrs = (C.c_void_p * S)(*[f.ctypes.data for f in frames_per_stream])
    steady = np.zeros(S, np.int64)
    hashes = np.zeros((S, nf, 2), np.uint64)
    nblobs = np.zeros((S, nf), np.int32)
    blobs = np.zeros((S, nf, bcap), BLOB_DTYPE)
    logs = np.zeros((S, lcap), LOG_DTYPE)
    nlog = np.zeros(S, np.int64)
    rc = L.ref_run_streams_detail(S, threads, w, h, ch, ptrs, nf, C.byref(mcfg), C.byref(scfg), C.byref(tcfg),
                                  steady.ctypes.data, hashes.ctypes.data, nblobs.ctypes.data, blobs.ctypes.data,
                                  bcap, logs.ctypes.data, lcap, nlog.ctypes.data)
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    out = []
    for s in range(S):
        k = int(steady[s])
        assert nlog[s] <= lcap, "raise lcap"
        out.append(dict(hashes=hashes[s, :k], nblobs=nblobs[s, :k], blobs=blobs[s, :k], log=logs[s, :nlog[s]]))
    return out


# ---------------------------------------------------------------------------
# object wrappers with one interface over both CPU checkers
# ---------------------------------------------------------------------------
class CpuMotion:
    def __init__(self, cfg: MOTION_CFG, w: int, h: int, impl: str = "orc"):
        self.impl, self.w, self.h = impl, w, h
        self.L = orc_lib() if impl == "orc" else ref_lib()
        self.cfg = cfg
        self.h_ = (self.L.orc_motion_create if impl == "orc" else self.L.ref_motion_create)(C.byref(cfg), w, h)
        if not self.h_:
            raise RuntimeError("motion create failed")

    def push(self, gray: np.ndarray):
        out = np.zeros(self.w * self.h, np.uint8)
        g = np.ascontiguousarray(gray, dtype=np.uint8)
        if self.impl == "orc":
            has = self.L.orc_motion_push(self.h_, g.ctypes.data, out.ctypes.data)
        else:
            hm = C.c_int(0)
            rc = self.L.ref_motion_push(self.h_, g.ctypes.data, self.w, self.h, 1, 0, out.ctypes.data, C.byref(hm))
            if rc:
                raise RuntimeError(self.L.ref_last_error().decode())
            has = hm.value
        return out if has else None

    def background(self):
        out = np.zeros(self.w * self.h, np.uint8)
        if self.impl == "orc":
            self.L.orc_motion_background(self.h_, out.ctypes.data)
        else:
            if self.L.ref_motion_background(self.h_, out.ctypes.data):
                raise RuntimeError(self.L.ref_last_error().decode())
        return out

    def __del__(self):
        try:
            (self.L.orc_motion_destroy if self.impl == "orc" else self.L.ref_motion_destroy)(self.h_)
        except Exception:
            pass


def cpu_label(mask: np.ndarray, w: int, h: int, conn: int = 1, min_area: int = 4, impl: str = "orc",
              n_blocks: int = 4, sequential: bool = False, want_pixels: bool = False):
    """-> (labels int32[w*h], blobs structured array, pixels or None)"""
    m = np.ascontiguousarray(mask, dtype=np.uint8)
    labels = np.zeros(w * h, np.int32)
    cap = w * h // 2 + 2
    blobs = (BLOB * cap)()
    pixels = np.zeros(int(np.count_nonzero(m)) + 1, np.int64) if want_pixels else None
    pp = pixels.ctypes.data if want_pixels else None
    if impl == "orc":
        n = orc_lib().orc_label(m.ctypes.data, w, h, conn, min_area, labels.ctypes.data, blobs, cap, pp)
    else:
        cfg = SEG_CFG(n_blocks, conn, min_area)
        nn = C.c_int(0)
        rc = ref_lib().ref_label(m.ctypes.data, w, h, C.byref(cfg), int(sequential), 1, labels.ctypes.data, blobs,
                                 cap, C.byref(nn), pp)
        if rc:
            raise RuntimeError(ref_lib().ref_last_error().decode())
        n = nn.value
    return labels, blobs_to_array(blobs, n), (pixels[:int(np.count_nonzero(labels))] if want_pixels else None)


WARP_ERRORS = {1: "homography has a non-finite entry", 2: "homography is not normalizable (h[2][2] = 0)",
               3: "homography is not invertible"}


def cpu_warp_frame(frame, w, h, ch, hom, impl="orc"):
    """warp_frame -> uint8[w*h*ch]; ValueError(message) on InvalidArgument."""
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    hm = np.ascontiguousarray(hom, dtype=np.float64).reshape(9)
    out = np.zeros(w * h * ch, np.uint8)
    if impl == "orc":
        rc = orc_lib().orc_warp_frame(f.ctypes.data, w, h, ch, hm.ctypes.data, out.ctypes.data)
        if rc:
            raise ValueError(WARP_ERRORS[rc])
    else:
        if ref_lib().ref_warp_frame(f.ctypes.data, w, h, ch, hm.ctypes.data, out.ctypes.data):
            raise ValueError(ref_lib().ref_last_error().decode())
    return out


def ref_stream_detect(frames, w, h, ch, homs, cfg: MOTION_CFG):
    """The reference's stream_detect (motion.hpp:260-282) -> masks [n-W+1, w*h]."""
    fr = np.ascontiguousarray(frames, dtype=np.uint8)
    n = fr.shape[0]
    hm = None if homs is None else np.ascontiguousarray(homs, dtype=np.float64)
    out = np.zeros((max(1, n - cfg.window + 1), w * h), np.uint8)
    nm = C.c_int(0)
    if ref_lib().ref_stream_detect(fr.ctypes.data, n, w, h, ch, None if hm is None else hm.ctypes.data,
                                   C.byref(cfg), out.ctypes.data, C.byref(nm)):
        raise ValueError(ref_lib().ref_last_error().decode())
    return out[:nm.value]


def cpu_blob_features(labels, w, h, frame, fw, fh, ch, blobs, impl="orc"):
    """extract_blob_features -> (mean_intensity[n], aspect[n]); raises
    ValueError on the reference's InvalidArgument (size mismatch)."""
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    f = np.ascontiguousarray(frame, dtype=np.uint8)
    b = np.ascontiguousarray(blobs)
    n = len(b)
    mean, aspect = np.zeros(max(n, 1)), np.zeros(max(n, 1))
    L = orc_lib() if impl == "orc" else ref_lib()
    fn = L.orc_blob_features if impl == "orc" else L.ref_blob_features
    rc = fn(lab.ctypes.data, w, h, f.ctypes.data, fw, fh, ch, b.ctypes.data if n else None, n, mean.ctypes.data,
            aspect.ctypes.data)
    if rc:
        raise ValueError(L.ref_last_error().decode() if impl != "orc" else "label image dimensions do not match frame")
    return mean[:n], aspect[:n]


class CpuTracker:
    def __init__(self, cfg: TRACKER_CFG, impl: str = "orc"):
        self.impl = impl
        self.L = orc_lib() if impl == "orc" else ref_lib()
        self.k = cfg.k_clusters
        self.h_ = (self.L.orc_tracker_create if impl == "orc" else self.L.ref_tracker_create)(C.byref(cfg))

    def process(self, frame: np.ndarray, w: int, h: int, ch: int, blobs):
        f = np.ascontiguousarray(frame, dtype=np.uint8)
        arr = (BLOB * max(1, len(blobs)))()
        for i, b in enumerate(blobs):
            arr[i] = BLOB(*[int(b[f_]) for f_ in ("label", "area", "x_min", "y_min", "x_max", "y_max")],
                          float(b["cx"]), float(b["cy"]))
        fn = self.L.orc_tracker_process if self.impl == "orc" else self.L.ref_tracker_process
        rc = fn(self.h_, f.ctypes.data, w, h, ch, arr, len(blobs))
        if self.impl == "ref" and rc:
            raise RuntimeError(self.L.ref_last_error().decode())

    def tracks(self):
        n = (self.L.orc_tracker_num_tracks if self.impl == "orc" else self.L.ref_tracker_num_tracks)(self.h_)
        arr = (TRACK * max(1, n))()
        (self.L.orc_tracker_tracks if self.impl == "orc" else self.L.ref_tracker_tracks)(self.h_, arr)
        return [arr[i] for i in range(n)]

    def track_model(self, i):
        c = np.zeros(self.k * 3)
        q = np.zeros(self.k)
        (self.L.orc_tracker_track_model if self.impl == "orc" else self.L.ref_tracker_track_model)(
            self.h_, i, c.ctypes.data, q.ctypes.data)
        return c.reshape(-1, 3), q

    def log(self):
        n = (self.L.orc_tracker_log_size if self.impl == "orc" else self.L.ref_tracker_log_size)(self.h_)
        arr = (LOGE * max(1, n))()
        (self.L.orc_tracker_log if self.impl == "orc" else self.L.ref_tracker_log)(self.h_, arr)
        return log_to_array(arr, n)

    def __del__(self):
        try:
            (self.L.orc_tracker_destroy if self.impl == "orc" else self.L.ref_tracker_destroy)(self.h_)
        except Exception:
            pass


def orc_frames(clip, n=None):
    """Frames of a synth Clip through the oracle restatement (synth.hpp)."""
    L = orc_lib()
    si, sd = clip.shape_arrays()
    si = np.array(si, np.int32)
    sd = np.array(sd, np.float64)
    s = L.orc_synth_create(clip.width, clip.height, clip.channels, clip.background, len(clip.shapes), si.ctypes.data,
                           sd.ctypes.data, clip.seed)
    n = clip.n_frames if n is None else n
    fb = clip.width * clip.height * clip.channels
    out = np.zeros((n, fb), np.uint8)
    rects = np.zeros((n, len(clip.shapes), 4), np.int32)
    try:
        for t in range(n):
            if L.orc_synth_next(s, out[t].ctypes.data, rects[t].ctypes.data) != 0:
                raise ValueError(f"shape leaves frame bounds at frame {t}")
    finally:
        L.orc_synth_destroy(s)
    return out, rects


def ref_frames(clip, n=None):
    L = ref_lib()
    si, sd = clip.shape_arrays()
    si = np.array(si, np.int32)
    sd = np.array(sd, np.float64)
    n = clip.n_frames if n is None else n
    fb = clip.width * clip.height * clip.channels
    out = np.zeros((n, fb), np.uint8)
    rects = np.zeros((n, len(clip.shapes), 4), np.int32)
    # synth_frames validates every frame of the clip; generate n frames
    rc = L.ref_synth(clip.width, clip.height, clip.channels, clip.background, len(clip.shapes), si.ctypes.data,
                     sd.ctypes.data, n, clip.seed, out.ctypes.data, rects.ctypes.data)
    if rc:
        raise RuntimeError(L.ref_last_error().decode())
    return out, rects


def grayscale(frame: np.ndarray, n_px: int) -> np.ndarray:
    out = np.zeros(n_px, np.uint8)
    orc_lib().orc_grayscale(np.ascontiguousarray(frame).ctypes.data, n_px, out.ctypes.data)
    return out


def run_pipeline_cpu(clip, frames, mcfg: MOTION_CFG, scfg: SEG_CFG, tcfg: TRACKER_CFG, impl="orc", n=None):
    """run_vision restated frame by frame (harness.hpp:412-450):
    push(gray) -> label_blocked -> Tracker::process.  Returns per-frame
    (mask, labels, blobs) for frames with a mask, and the track log."""
    w, h, ch = clip.width, clip.height, clip.channels
    n = len(frames) if n is None else n
    mot = CpuMotion(mcfg, w, h, impl)
    trk = CpuTracker(tcfg, impl)
    out = []
    for t in range(n):
        f = frames[t]
        g = f if ch == 1 else grayscale(f, w * h)
        m = mot.push(g)
        if m is None:
            continue
        lab, blobs, _ = cpu_label(m, w, h, scfg.connectivity, scfg.min_area, impl, scfg.n_blocks)
        trk.process(f, w, h, ch, blobs)
        out.append((t, m, lab, blobs))
    return out, trk.log(), trk

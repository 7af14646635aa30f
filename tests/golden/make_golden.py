"""Generates tests/golden/*.npz from the UNMODIFIED reference.

Runs the reference headers (compiled by oracle/Makefile into
oracle/_ref/libteamrec_ref.so from /root/reference/proj/include) on the
cases below and stores compact results: per-frame SHA-256 digests of the
masks and label images, the blob tables and the full track logs.  Re-run
after changing a case:

    make -C oracle && python tests/golden/make_golden.py

Cases:
  c1_pipeline       recipe C1, frames 0..159, default configs
  c2_pipeline       recipe C2 (UC-Teamwork-like), frames 0..139
  harness_vision    harness_test.cpp:377-389 clip (48x36 RGB, W=9)
  bench_vision      bench_run's clip (harness.hpp:571-581, 96x72 RGB, W=91)
  two_squares       tracking_test.cpp:249-270 clip, TrackerConfig k=4 seed=7
  acceptance6       acceptance.cpp:344-358 clip (criterion 6), default tracker
  retire            tracking_test.cpp:343-372 (lost tracks retire after 5)
  random_ccl        200 random 32x32 masks (seed 303, acceptance.cpp:139-171)
"""
from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import Clip, Rng, Shape, bench_vision_clip, harness_vision_clip, recipe  # noqa: E402
from tests import _oracle as O  # noqa: E402


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def two_squares_clip() -> Clip:
    red, yellow, blue = (255, 0, 0), (255, 255, 0), (0, 0, 255)
    shapes = [Shape(9, 9, red, 4, 4, 0.5, 0.25), Shape(5, 5, yellow, 6, 6, 0.5, 0.25),
              Shape(9, 9, blue, 48, 32, -0.5, 0.0), Shape(5, 5, red, 50, 34, -0.5, 0.0)]
    return Clip(64, 48, 3, 0, shapes, 30, 0, "two_squares")


def acceptance6_clip() -> Clip:
    span = 29.0
    shapes = [Shape(9, 9, (230, 40, 40), 4.0, 6.0, (46.0 - 4.0) / span, (12.0 - 6.0) / span),
              Shape(8, 8, (40, 60, 230), 52.0, 36.0, (6.0 - 52.0) / span, (30.0 - 36.0) / span)]
    return Clip(64, 48, 3, 0, shapes, 30, 606, "acceptance6")


def random_mask(w, h, density, rng: Rng) -> np.ndarray:
    """oracle::random_mask (tests/oracles.hpp:90-94)."""
    return np.array([1 if rng.uniform() < density else 0 for _ in range(w * h)], np.uint8)


def pipeline_case(clip: Clip, n: int, mcfg: MOTION_CFG, impl: str = "ref"):
    frames, _ = O.ref_frames(clip, n) if impl == "ref" else O.orc_frames(clip, n)
    out, log, _ = O.run_pipeline_cpu(clip, frames, mcfg, SEG_CFG(), TRACKER_CFG(), impl)
    steady = np.array([t for t, *_ in out], np.int32)
    mask_sha = np.array([sha(m) for _, m, _, _ in out])
    label_sha = np.array([sha(l_) for _, _, l_, _ in out])
    nblobs = np.array([len(b) for *_, b in out], np.int32)
    blobs = np.concatenate([b for *_, b in out]) if out else np.zeros(0)
    return dict(steady=steady, mask_sha=mask_sha, label_sha=label_sha, nblobs=nblobs, blobs=blobs, log=log,
                frames_sha=np.array([sha(f) for f in frames]))


def tracker_case(clip: Clip, tcfg: TRACKER_CFG, min_area=4):
    frames, rects = O.ref_frames(clip)
    trk = O.CpuTracker(tcfg, "ref")
    w, h = clip.width, clip.height
    for t in range(clip.n_frames):
        # blobs of the generator's union mask (tracking_test.cpp blobs_of)
        m = np.zeros(w * h, np.uint8)
        for (ix, iy, rw, rh) in rects[t]:
            mm = m.reshape(h, w)
            mm[iy:iy + rh, ix:ix + rw] = 1
        _, blobs, _ = O.cpu_label(m, w, h, 1, min_area, "ref", sequential=True)
        trk.process(frames[t], w, h, clip.channels, blobs)
    return dict(log=trk.log(), frames_sha=np.array([sha(f) for f in frames]))


def blob_features_case(trials: int = 40):
    """extract_blob_features (segmentation.hpp:268-291) on random masks and
    frames through the reference: ragged sizes, 4/8-connectivity, gray and
    RGB.  Inputs and outputs flattened with offsets."""
    rng = np.random.default_rng(11)
    d = {k: [] for k in ("dims", "masks", "frames", "labels", "blobs", "mean", "aspect")}
    for trial in range(trials):
        w, h = int(rng.integers(1, 49)), int(rng.integers(1, 49))
        ch = 1 if trial % 3 else 3
        conn = int(trial % 2)
        min_area = int(rng.integers(1, 5))
        m = (rng.random(w * h) < rng.uniform(0.1, 0.8)).astype(np.uint8)
        f = rng.integers(0, 256, size=w * h * ch, dtype=np.uint8)
        lab, blobs, _ = O.cpu_label(m, w, h, conn, min_area, "ref", n_blocks=1)
        mean, aspect = O.cpu_blob_features(lab, w, h, f, w, h, ch, blobs, "ref")
        d["dims"].append((w, h, ch, conn, min_area, len(blobs)))
        d["masks"].append(m)
        d["frames"].append(f)
        d["labels"].append(lab)
        d["blobs"].append(np.frombuffer(blobs.tobytes(), np.uint8))
        d["mean"].append(mean)
        d["aspect"].append(aspect)
    out = {"dims": np.array(d["dims"], np.int32)}
    for k in ("masks", "frames", "labels", "blobs", "mean", "aspect"):
        out[k] = np.concatenate(d[k]) if d[k] else np.zeros(0)
    return out


def _random_homography(rng, kind):
    if kind == 0:
        return np.eye(3)
    if kind == 1:  # fractional translation
        h = np.eye(3)
        h[0, 2], h[1, 2] = rng.uniform(-6, 6), rng.uniform(-6, 6)
        return h
    if kind == 2:  # rotation + scale + translation
        a, sc = rng.uniform(-0.4, 0.4), rng.uniform(0.7, 1.4)
        return np.array([[sc * np.cos(a), -sc * np.sin(a), rng.uniform(-5, 5)],
                         [sc * np.sin(a), sc * np.cos(a), rng.uniform(-5, 5)], [0.0, 0.0, 1.0]])
    if kind == 3:  # projective
        h = np.eye(3) + rng.uniform(-0.05, 0.05, size=(3, 3))
        h[2, 0], h[2, 1] = rng.uniform(-0.01, 0.01), rng.uniform(-0.01, 0.01)
        h[2, 2] = rng.uniform(0.8, 1.2)
        return h
    h = np.eye(3)  # everything maps off the source plane
    h[0, 2] = 1e4
    return h


def warp_case(trials: int = 40):
    """warp_frame (motion.hpp:81-119) through the reference on random frames
    and homographies (identity, sub-pixel translation, rotation/scale,
    projective, off-plane), gray and RGB; plus stream_detect (:260-282) with
    per-frame homographies on a small clip."""
    rng = np.random.default_rng(21)
    dims, frames, homs, outs = [], [], [], []
    for trial in range(trials):
        w, h, ch = int(rng.integers(1, 65)), int(rng.integers(1, 65)), 1 if trial % 3 else 3
        f = rng.integers(0, 256, size=w * h * ch, dtype=np.uint8)
        hm = _random_homography(rng, trial % 5)
        dims.append((w, h, ch))
        frames.append(f)
        homs.append(hm.reshape(9))
        outs.append(O.cpu_warp_frame(f, w, h, ch, hm, "ref"))
    # stream_detect on a panning 48x36 clip, W = 9
    clip = harness_vision_clip()
    n = 20
    cf, _ = O.ref_frames(clip, n)
    sh = np.stack([np.array([[1, 0.02 * t, 0.7 * t], [-0.02 * t, 1, -0.4 * t], [0, 0, 1]], np.float64).reshape(9)
                   for t in range(n)])
    mcfg = MOTION_CFG(window=9)
    mcfg.warp = 1
    masks = O.ref_stream_detect(cf, clip.width, clip.height, clip.channels, sh, mcfg)
    return dict(dims=np.array(dims, np.int32), frames=np.concatenate(frames), homs=np.array(homs),
                outs=np.concatenate(outs), stream_frames=cf, stream_homs=sh, stream_masks=masks)


PNM_CASES = [
    b"P5\n3 2\n255\n" + bytes(range(6)),
    b"P6 2 2 255 " + bytes(range(12)),
    b"P5\n# a comment\n  4 1 # trailing\n255\n" + b"abcd",
    b"P5\t1\r1\x0b255\n\x07extra",
    b"P2 3 2 255 " + bytes(6),
    b"P5 3 2 65535 " + bytes(12),
    b"P5 3x 2 255 " + bytes(6),
    b"P5 0 2 255 ",
    b"P5 -3 2 255 ",
    b"P5 3 2",
    b"P5 3 2 255 " + bytes(5),
    b"",
    b"# only a comment",
    b"P6 +2 1 255 " + bytes(6),
    b"P5 99999999999 1 255 ",
]


def io_case():
    """decode_pnm (frame.hpp:152-175) and the track-log text format
    (tracking.hpp:247-277) through the reference."""
    L = O.ref_lib()
    import ctypes as C
    dims, px, errs = [], [], []
    for b in PNM_CASES:
        buf = np.frombuffer(b, np.uint8) if b else np.zeros(1, np.uint8)
        w, h, c = C.c_int(0), C.c_int(0), C.c_int(0)
        out = np.zeros(256, np.uint8)
        rc = L.ref_decode_pnm(buf.ctypes.data, len(b), b"<memory>", C.byref(w), C.byref(h), C.byref(c),
                              out.ctypes.data, out.size)
        if rc:
            dims.append((0, 0, 0))
            errs.append(L.ref_last_error().decode())
            px.append(np.zeros(0, np.uint8))
        else:
            dims.append((w.value, h.value, c.value))
            errs.append("")
            px.append(out[:w.value * h.value * c.value].copy())
    log = np.load(os.path.join(HERE, "acceptance6.npz"))["log"]
    text = C.create_string_buffer(1 << 20)
    n = L.ref_format_track_log(log.ctypes.data, len(log), text, len(text))
    return dict(pnm_dims=np.array(dims, np.int32), pnm_pixels=np.concatenate(px), pnm_errors=np.array(errs),
                log=log, log_text=np.frombuffer(text.raw[:n], np.uint8))


def main():
    if not O.ref_available():
        sys.exit("oracle/_ref/libteamrec_ref.so missing: run `make -C oracle` where /root/reference exists")
    out = {}
    if "blob_features" in sys.argv[1:]:  # only the extract_blob_features fixture
        out["blob_features"] = blob_features_case()
    if "warp" in sys.argv[1:]:  # only the warp_frame / stream_detect fixture
        out["warp"] = warp_case()
    if "io" in sys.argv[1:]:  # only the PNM / track-log text fixture
        out["io"] = io_case()
    if out:
        for name, d in out.items():
            np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
            print(name, {k: getattr(v, "shape", None) for k, v in d.items()})
        return
    out["c1_pipeline"] = pipeline_case(recipe("C1"), 160, MOTION_CFG())
    out["c2_pipeline"] = pipeline_case(recipe("C2"), 140, MOTION_CFG())
    out["harness_vision"] = pipeline_case(harness_vision_clip(), 29, MOTION_CFG(window=9))
    bc = bench_vision_clip()
    out["bench_vision"] = pipeline_case(bc, bc.n_frames, MOTION_CFG())
    out["two_squares"] = tracker_case(two_squares_clip(), TRACKER_CFG(k_clusters=4, seed=7))
    out["acceptance6"] = tracker_case(acceptance6_clip(), TRACKER_CFG())
    # random CCL masks, acceptance.cpp:139-171 (density 0.25 + 0.5*u, conn alternating, min_area 1)
    rng = Rng(303)
    masks, labels_sha, nb, conns = [], [], [], []
    for trial in range(200):
        density = 0.25 + 0.5 * rng.uniform()
        m = random_mask(32, 32, density, rng)
        conn = 1 if trial % 2 else 0
        lab, blobs, _ = O.cpu_label(m, 32, 32, conn, 1, "ref", n_blocks=4)
        masks.append(m)
        labels_sha.append(sha(lab))
        nb.append(len(blobs))
        conns.append(conn)
    out["random_ccl"] = dict(masks=np.array(masks), label_sha=np.array(labels_sha), nblobs=np.array(nb),
                             conn=np.array(conns))
    out["blob_features"] = blob_features_case()
    out["warp"] = warp_case()
    out["io"] = io_case()
    for name, d in out.items():
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **d)
        print(name, {k: getattr(v, "shape", None) for k, v in d.items()})


if __name__ == "__main__":
    main()

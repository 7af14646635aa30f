"""GPU parity: motion detector and connected components vs the oracle.

Every comparison is bit-exact (masks, labels, blob tables incl. the fp64
centroids).  Cases follow the reference's own tests (motion_test.cpp,
segmentation_test.cpp, acceptance.cpp:139-171) plus edge shapes (ragged
tiles, 1-pixel-wide frames, all-background / all-foreground) and full-size
frames of the benchmark recipes.
"""
import os

import numpy as np
import pytest

from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG
from paper_1310_3322_b200.synth import Rng, recipe
from tests import _oracle as O
from tests.golden.make_golden import random_mask, sha

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run_motion_pair(trb, cfg, w, h, frames):
    g = trb.MotionDetector(cfg, w, h)
    o = O.CpuMotion(cfg, w, h, "orc")
    n = 0
    for i, f in enumerate(frames):
        a = g.push(f, index=i)
        b = o.push(f)
        assert (a is None) == (b is None), f"frame {i}: mask presence differs"
        if a is not None:
            assert np.array_equal(a, b), f"frame {i}: mask differs"
            n += 1
    if n:
        assert np.array_equal(g.background(), o.background())
    return n


@pytest.mark.parametrize("window", [2, 5, 91, 257, 300])
def test_motion_random_frames(gpu, window):
    rng = np.random.default_rng(window)
    w, h = 37, 23  # ragged: px not a multiple of 16
    frames = [rng.integers(0, 256, w * h, dtype=np.uint8) for _ in range(window + 6)]
    assert run_motion_pair(gpu, MOTION_CFG(window=window, threshold=40), w, h, frames) == 7


@pytest.mark.parametrize("bins", [2, 7, 32, 256])
def test_motion_mode_method(gpu, bins):
    rng = np.random.default_rng(bins)
    w, h = 33, 17
    frames = [(rng.integers(0, 4, w * h) * 70).astype(np.uint8) for _ in range(12)]
    run_motion_pair(gpu, MOTION_CFG(method=1, window=9, bins=bins, threshold=20), w, h, frames)


def test_motion_known_answers(gpu):
    # motion_test.cpp:238-250: 91 constant frames then one change
    d = gpu.MotionDetector(MOTION_CFG(window=91), 4, 4)
    masks = []
    for i in range(92):
        f = np.full(16, 60, np.uint8)
        if i == 91:
            f[9] = 255
            f[3] = 255
        m = d.push(f, index=i)
        if m is not None:
            masks.append(m)
    assert len(masks) == 2 and masks[0].sum() == 0 and masks[1].sum() == 2 and masks[1][9] and masks[1][3]
    # :54-66 / :68-73 via background()
    for vals, method, want in (([10, 10, 250], 0, 90), ([10, 10, 250], 1, 10), ([1, 2], 0, 2),
                               ([2, 4, 250, 252], 1, 3)):
        d = gpu.MotionDetector(MOTION_CFG(method=method, window=len(vals)), 1, 1)
        for v in vals:
            d.push(np.array([v], np.uint8))
        assert int(d.background()[0]) == want


def test_motion_errors(gpu):
    d = gpu.MotionDetector(MOTION_CFG(window=5), 8, 8)
    with pytest.raises(gpu.InvalidArgument, match="expects grayscale"):
        d.push(np.zeros(64 * 3, np.uint8), channels=3)
    with pytest.raises(gpu.InvalidArgument, match="frame 7 dimensions do not match detector"):
        d.push(np.zeros(63, np.uint8), width=9, height=7, index=7)
    with pytest.raises(gpu.InvalidArgument, match="before the window fills"):
        d.background()
    with pytest.raises(gpu.ConfigError):
        gpu.MotionDetector(MOTION_CFG(window=1), 8, 8)
    with pytest.raises(gpu.InvalidArgument, match="positive frame dimensions"):
        gpu.MotionDetector(MOTION_CFG(window=5), 0, 8)


@pytest.mark.parametrize("name,n", [("C1", 130), ("C2", 120)])
def test_motion_recipes(gpu, name, n):
    clip = recipe(name)
    frames, _ = O.orc_frames(clip, n)
    run_motion_pair(gpu, MOTION_CFG(), clip.width, clip.height, frames)


@pytest.mark.parametrize("op", [1, 2, 3, 4])
def test_morphology_vs_oracle(gpu, op):
    """3x3 morphology (not in the reference): parity vs the oracle's
    restatement of the stated border rule."""
    clip = recipe("C2")
    frames, _ = O.orc_frames(clip, 100)
    run_motion_pair(gpu, MOTION_CFG(morph=op), clip.width, clip.height, frames)


# ------------------------------------------------------------------ CCL
def check_label(trb, m, w, h, conn, min_area, n_blocks=4, pixels=False):
    lab = trb.label_blocked(m, w, h, SEG_CFG(n_blocks, conn, min_area), want_pixels=pixels)
    want_l, want_b, want_p = O.cpu_label(m, w, h, conn, min_area, "orc", want_pixels=pixels)
    assert np.array_equal(lab.labels, want_l)
    assert lab.blobs.tobytes() == want_b.tobytes()
    if pixels:
        assert np.array_equal(lab._pixels, want_p)
    return lab


def test_ccl_random_masks_golden(gpu):
    """acceptance.cpp:139-171 masks (seed 303): labels == the reference's."""
    g = np.load(os.path.join(GOLD, "random_ccl.npz"))
    for m, want, nb, conn in zip(g["masks"], g["label_sha"], g["nblobs"], g["conn"]):
        for n_blocks in (1, 4, 16):
            lab = gpu.label_blocked(m, 32, 32, SEG_CFG(n_blocks, int(conn), 1))
            assert sha(lab.labels) == want and len(lab.blobs) == nb


@pytest.mark.parametrize("seed,density", [(301, 0.45), (302, 0.4), (303, 0.5), (304, 0.5), (9, 0.1), (10, 0.9)])
def test_ccl_random_masks_vs_oracle(gpu, seed, density):
    rng = Rng(seed)
    for it in range(12):
        w, h = [(32, 32), (45, 70), (100, 33), (64, 64)][it % 4]
        m = random_mask(w, h, density, rng)
        for conn in (0, 1):
            for min_area in (1, 4):
                check_label(gpu, m, w, h, conn, min_area, pixels=(it == 0))


@pytest.mark.parametrize("w,h", [(1, 1), (1, 200), (200, 1), (31, 33), (33, 31), (1000, 3)])
def test_ccl_edge_shapes(gpu, w, h):
    rng = np.random.default_rng(w * 1000 + h)
    for density in (0.0, 0.3, 0.7, 1.0):
        m = (rng.random(w * h) < density).astype(np.uint8)
        for conn in (0, 1):
            n_blocks = 1 if min(w, h) < 2 else 4
            check_label(gpu, m, w, h, conn, 1, n_blocks=n_blocks)


def test_ccl_checkerboard_and_stripes(gpu):
    w, h = 128, 96
    y, x = np.mgrid[0:h, 0:w]
    for m in ((x + y) % 2, (x % 3 == 0), (y % 2 == 0), ((x // 5 + y // 7) % 2), np.ones((h, w))):
        m = m.astype(np.uint8).reshape(-1)
        for conn in (0, 1):
            check_label(gpu, m, w, h, conn, 1)
    # one spiral component snaking through every tile
    s = np.zeros((h, w), np.uint8)
    s[::4, :] = 1
    for r in range(0, h - 4, 4):
        s[r:r + 4, (w - 1) if (r // 4) % 2 == 0 else 0] = 1
    check_label(gpu, s.reshape(-1), w, h, 0, 1)
    lab = gpu.label_blocked(s.reshape(-1), w, h, SEG_CFG(4, 0, 1))
    assert len(lab.blobs) == 1


def test_ccl_known_answers_and_errors(gpu):
    m = np.zeros(25, np.uint8)
    for x, y in [(4, 0), (0, 2), (1, 2), (3, 4)]:
        m[y * 5 + x] = 1
    lab = gpu.label_sequential(m, 5, 5, SEG_CFG(4, 0, 1))
    assert lab.label_at(4, 0) == 1 and lab.label_at(0, 2) == 2 and lab.label_at(1, 2) == 2
    assert lab.label_at(3, 4) == 3
    with pytest.raises(gpu.ConfigError, match="n_blocks=7 does not tile a 4x4 image"):
        gpu.label_blocked(np.zeros(16, np.uint8), 4, 4, SEG_CFG(7, 1, 1))
    with pytest.raises(gpu.ConfigError):
        gpu.label_blocked(np.zeros(16, np.uint8), 4, 4, SEG_CFG(64, 1, 1))
    gpu.label_blocked(np.zeros(16, np.uint8), 4, 4, SEG_CFG(16, 1, 1))


@pytest.mark.parametrize("name", ["C3", "C4"])
def test_ccl_full_size_recipe_masks(gpu, name):
    """Full-size 1080p / 4K masks straight from the recipes' ground-truth
    rectangles (plus noise): labels and blobs bit-identical."""
    clip = recipe(name)
    rects = clip.all_rects(5)
    rng = np.random.default_rng(3)
    for t in (0, 4):
        m = np.zeros((clip.height, clip.width), np.uint8)
        for ix, iy, rw, rh in rects[t]:
            m[iy:iy + rh, ix:ix + rw] = 1
        m = m.reshape(-1)
        noise = rng.random(m.size) < 0.001
        m = (m ^ noise).astype(np.uint8)
        check_label(gpu, m, clip.width, clip.height, 1, 4)


# ---------------------------------------------- extract_blob_features (§8(f) 2)
def test_blob_features_golden(gpu):
    """Device labels -> device extract_blob_features vs the reference's
    values (tests/golden/blob_features.npz): ragged sizes, 4/8-conn, gray/RGB."""
    g = np.load(os.path.join(GOLD, "blob_features.npz"))
    om = oa = ol = 0
    for w, h, ch, conn, min_area, nb in g["dims"]:
        m, f = g["masks"][om:om + w * h], g["frames"][oa:oa + w * h * ch]
        lab = gpu.label_blocked(m, w, h, SEG_CFG(1, conn, min_area))
        assert lab.labels.tobytes() == g["labels"][om:om + w * h].tobytes()
        mean, aspect = gpu.extract_blob_features(lab.labels, w, h, f, w, h, ch, lab.blobs)
        assert mean.tobytes() == g["mean"][ol:ol + nb].tobytes()
        assert aspect.tobytes() == g["aspect"][ol:ol + nb].tobytes()
        om, oa, ol = om + w * h, oa + w * h * ch, ol + nb


def test_blob_features_known_answers_and_errors(gpu):
    from paper_1310_3322_b200.api import InvalidArgument
    m = np.zeros(16, np.uint8)
    f = np.zeros(48, np.uint8)
    m[5] = 1
    f[15] = 255  # pure red at (1, 1)
    lab = gpu.label_blocked(m, 4, 4, SEG_CFG(1, 1, 1))
    mean, aspect = gpu.extract_blob_features(lab.labels, 4, 4, f, 4, 4, 3, lab.blobs)
    assert mean[0] == float((77 * 255 + 128) // 256) and aspect[0] == 1.0
    empty = gpu.label_blocked(np.zeros(16, np.uint8), 4, 4, SEG_CFG(1, 1, 1))
    assert len(gpu.extract_blob_features(empty.labels, 4, 4, np.zeros(16, np.uint8), 4, 4, 1, empty.blobs)[0]) == 0
    with pytest.raises(InvalidArgument, match="label image dimensions do not match frame"):
        gpu.extract_blob_features(lab.labels, 4, 4, np.zeros(20, np.uint8), 5, 4, 1, lab.blobs)


def test_blob_features_full_frame_vs_oracle(gpu):
    """A 1080p C3 mask with its frame: large blobs (long label runs, one
    atomic per run) vs the oracle."""
    clip = recipe("C3")
    frames, _ = O.orc_frames(clip, 100)
    mot = O.CpuMotion(MOTION_CFG(), clip.width, clip.height, "orc")
    m = None
    for t in range(92):
        m = mot.push(frames[t])
    lab = gpu.label_blocked(m, clip.width, clip.height, SEG_CFG())
    mean, aspect = gpu.extract_blob_features(lab.labels, clip.width, clip.height, frames[91], clip.width,
                                             clip.height, 1, lab.blobs)
    om, oa = O.cpu_blob_features(lab.labels, clip.width, clip.height, frames[91], clip.width, clip.height, 1,
                                 lab.blobs, "orc")
    assert len(mean) > 5
    assert mean.tobytes() == om.tobytes() and aspect.tobytes() == oa.tobytes()


# ---------------------------------------------------- warp_frame (§8(f) 4)
def test_warp_frame_golden(gpu):
    g = np.load(os.path.join(GOLD, "warp.npz"))
    of = 0
    for (w, h, ch), hm in zip(g["dims"], g["homs"]):
        n = w * h * ch
        out = gpu.warp_frame(g["frames"][of:of + n], w, h, ch, hm)
        assert out.tobytes() == g["outs"][of:of + n].tobytes()
        of += n


def test_warp_frame_errors_and_large(gpu):
    from paper_1310_3322_b200.api import InvalidArgument
    f = np.zeros(12, np.uint8)
    for hm, msg in [([[1, 0, np.inf], [0, 1, 0], [0, 0, 1]], "non-finite"),
                    ([[1, 0, 0], [0, 1, 0], [0, 0, 0.0]], "not normalizable"),
                    ([[1, 2, 0], [2, 4, 0], [0, 0, 1.0]], "not invertible")]:
        with pytest.raises(InvalidArgument, match=msg):
            gpu.warp_frame(f, 4, 3, 1, np.array(hm, np.float64))
    # a full 1080p frame under a projective homography vs the oracle
    rng = np.random.default_rng(3)
    fr = rng.integers(0, 256, size=1920 * 1080, dtype=np.uint8)
    hm = np.array([[0.98, 0.05, 12.3], [-0.04, 1.01, -7.7], [1e-5, -2e-5, 1.0]])
    assert gpu.warp_frame(fr, 1920, 1080, 1, hm).tobytes() == O.cpu_warp_frame(fr, 1920, 1080, 1, hm).tobytes()


@pytest.mark.parametrize("w,h", [(16, 1), (16, 17), (48, 36), (320, 240), (1920, 40), (17, 9), (100, 33), (1, 5)])
def test_morph_device_planes_vs_oracle(gpu, w, h):
    """trb_morph_device on several random 0/1 planes at once: the fused
    row-strip kernel (widths % 16 == 0, strips of 16 rows, 30-block warps)
    and the tiled two-pass fallback, every op, vs the oracle's orc_morph."""
    import ctypes as C
    import torch
    from paper_1310_3322_b200 import api
    rng = np.random.default_rng(w * 1000 + h)
    n = 3
    masks = [(rng.random((h, w)) < p).astype(np.uint8) for p in (0.5, 0.9, 0.1)]
    dev_in = torch.from_numpy(np.stack(masks)).cuda()
    for op in (1, 2, 3, 4):
        dev_out = torch.full_like(dev_in, 7)
        api.morph_device(dev_in.data_ptr(), dev_out.data_ptr(), w, h, n, op)
        torch.cuda.synchronize()
        got = dev_out.cpu().numpy()
        for k in range(n):
            want = np.zeros((h, w), np.uint8)
            O.orc_lib().orc_morph(masks[k].ctypes.data, w, h, op, want.ctypes.data)
            assert np.array_equal(got[k], want), (op, k)


@pytest.mark.parametrize("window,bins,levels", [(9, 7, 4), (9, 32, 9), (20, 2, 3), (91, 32, 6), (255, 16, 5),
                                                (256, 16, 5)])
def test_motion_mode_incremental_long_runs(gpu, window, bins, levels):
    """The incremental Mode state (per-bin counts / sums, mode bin; W <= 255)
    over long runs with many evictions, ties between bins and mode changes,
    every mask and the final background vs the oracle; W = 256 takes the
    ring re-read path."""
    rng = np.random.default_rng(window * 100 + bins)
    w, h = 29, 13
    step = 255 // (levels - 1)
    frames = []
    base = (rng.integers(0, levels, w * h) * step).astype(np.uint8)
    for i in range(window + 40):
        f = base.copy()
        flip = rng.random(w * h) < 0.35  # moving "objects": many pixels change bin, modes flip
        f[flip] = (rng.integers(0, levels, int(flip.sum())) * step).astype(np.uint8)
        if i % 7 == 0:
            base = f
        frames.append(f)
    assert run_motion_pair(gpu, MOTION_CFG(method=1, window=window, bins=bins, threshold=20), w, h, frames) == 41


def test_streams_mode_background_clip_vs_oracle(gpu):
    """Mode background through the batched handle (the incremental kernel)
    on a moving-blob clip, RGB and gray: masks, labels and track logs equal
    the oracle pipeline."""
    from paper_1310_3322_b200.abi import SEG_CFG, TRACKER_CFG
    from paper_1310_3322_b200.synth import harness_vision_clip, recipe
    from tests.golden.make_golden import sha
    for clip, n, mcfg in ((recipe("C1"), 130, MOTION_CFG(method=1, bins=32)),
                          (harness_vision_clip(), 29, MOTION_CFG(method=1, window=9, bins=16))):
        frames, _ = O.orc_frames(clip, n)
        st = gpu.Streams(1, clip.width, clip.height, clip.channels, mcfg, SEG_CFG(), TRACKER_CFG())
        got = []
        for t in range(n):
            st.step_host([frames[t]])
            if st.has_output:
                got.append((sha(st.mask(0)), sha(st.labels(0))))
        st.synchronize()
        out, log, _ = O.run_pipeline_cpu(clip, frames, mcfg, SEG_CFG(), TRACKER_CFG(), "orc")
        assert got == [(sha(m), sha(l_)) for _, m, l_, _ in out]
        assert st.log(0).tobytes() == log.tobytes()

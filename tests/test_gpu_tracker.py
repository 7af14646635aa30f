"""GPU parity: the device tracker (mean-shift with exact-order fp64 sums,
gating, spawn k-means, retirement, log) vs the oracle and the golden logs
of the unmodified reference.  Track logs are compared byte-for-byte, i.e.
every %.17g digit of every coordinate."""
import os

import numpy as np
import pytest

from paper_1310_3322_b200.abi import BLOB_DTYPE, MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import recipe
from tests import _oracle as O
from tests.golden.make_golden import acceptance6_clip, two_squares_clip

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_glibc_hypot_on_device(gpu):
    from paper_1310_3322_b200 import api
    rng = np.random.default_rng(2)
    n = 200000
    x = np.concatenate([rng.uniform(-4000, 4000, n), np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-1074, 1023, n))])
    y = np.concatenate([rng.uniform(-4000, 4000, n), np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-1074, 1023, n))])
    dev = api.selftest_hypot(x, y, on_device=True)
    L = O.orc_lib()
    want = np.array([L.orc_libm_hypot(a, b) for a, b in zip(x, y)])
    assert dev.tobytes() == want.tobytes()


def test_quantize_colors_vs_oracle(gpu):
    rng = np.random.default_rng(11)
    for trial in range(25):
        n = int(rng.integers(16, 3000))
        k = int(rng.integers(2, 17))
        levels = int(rng.integers(1, 20))
        px = (rng.integers(0, levels, size=(n, 3)) * (255 // max(1, levels - 1) if levels > 1 else 7)).astype(float)
        want = np.zeros(3 * k)
        O.orc_lib().orc_quantize_colors(px.ctypes.data, n, k, 20, trial * 7 + 1, want.ctypes.data)
        got = gpu.quantize_colors(px, k, 20, trial * 7 + 1)
        assert got.reshape(-1).tobytes() == want.tobytes(), trial


def test_quantize_colors_real_valued_vs_oracle(gpu):
    """Real-valued samples (tracking_test.cpp:95-121: noisy clumps, uniform
    random colours): the sequential device kernel, bit-identical centres."""
    rng = np.random.default_rng(5)
    clumps = np.array([[30, 30, 30], [200, 50, 50], [60, 220, 100]], float)
    cases = [(clumps[np.arange(60) % 3] + rng.uniform(-5.0, 5.0, (60, 3)), 3, 30, 11),
             (rng.uniform(0.0, 255.0, (40, 3)), 4, 20, 9),
             (rng.uniform(0.0, 255.0, (700, 3)), 16, 20, 123),
             (np.round(rng.uniform(0, 255, (300, 3))) + 0.5, 8, 20, 77),
             # duplicates -> empty clusters (farthest-point re-seed), many samples, large k
             (np.repeat(rng.uniform(0.0, 255.0, (5, 3)), 40, axis=0) + 0.25, 9, 20, 5),
             (rng.uniform(0.0, 255.0, (40000, 3)), 24, 15, 31),
             (clumps[np.arange(20000) % 3] + rng.normal(0.0, 3.0, (20000, 3)), 70, 10, 2)]
    for px, k, iters, seed in cases:
        px = np.ascontiguousarray(px)
        want = np.zeros(3 * k)
        O.orc_lib().orc_quantize_colors(px.ctypes.data, len(px), k, iters, seed, want.ctypes.data)
        got = gpu.quantize_colors(px, k, iters, seed)
        assert got.reshape(-1).tobytes() == want.tobytes(), (len(px), k)
        assert (gpu.quantize_colors(px, k, iters, seed) == got).all()  # deterministic


def test_quantize_degenerate_and_errors(gpu):
    px = np.tile([50.0, 60.0, 70.0], (10, 1))
    c = gpu.quantize_colors(px, 2, 20, 3)
    assert (c == [50, 60, 70]).all()
    with pytest.raises(gpu.InvalidArgument):
        gpu.quantize_colors(px, 1, 20, 3)
    with pytest.raises(gpu.InvalidArgument):
        gpu.quantize_colors(px[:1], 2, 20, 3)


def random_case(rng, big=False):
    if big:
        w, h = int(rng.integers(300, 700)), int(rng.integers(200, 500))
    else:
        w, h = int(rng.integers(8, 90)), int(rng.integers(8, 90))
    ch = int(rng.choice([1, 3]))
    levels = int(rng.integers(2, 6))
    f = (rng.integers(0, levels, size=w * h * ch) * (255 // (levels - 1))).astype(np.uint8)
    k = int(rng.integers(2, 17))
    cen = rng.integers(0, levels, size=3 * k).astype(np.float64) * (255 // (levels - 1)) + rng.random(3 * k) * 3
    cx, cy = float(rng.uniform(-2, w + 2)), float(rng.uniform(-2, h + 2))
    tw, th = int(rng.integers(3, max(4, w))), int(rng.integers(3, max(4, h)))
    return w, h, ch, f, k, cen, cx, cy, tw, th


@pytest.mark.parametrize("big", [False, True])
def test_histogram_vs_oracle(gpu, big):
    rng = np.random.default_rng(21 + big)
    for trial in range(30 if not big else 8):
        w, h, ch, f, k, cen, cx, cy, tw, th = random_case(rng, big)
        want = np.zeros(k)
        ok = O.orc_lib().orc_histogram(f.ctypes.data, w, h, ch, cx, cy, tw, th, cen.ctypes.data, k, 1, want.ctypes.data)
        if not ok:
            with pytest.raises(gpu.InvalidArgument):
                gpu.histogram(f, w, h, ch, cx, cy, tw, th, cen)
            continue
        got = gpu.histogram(f, w, h, ch, cx, cy, tw, th, cen)
        assert got.tobytes() == want.tobytes(), trial


@pytest.mark.parametrize("big", [False, True])
def test_meanshift_vs_oracle(gpu, big):
    import ctypes as C
    rng = np.random.default_rng(31 + big)
    tested = 0
    for trial in range(60 if not big else 10):
        w, h, ch, f, k, cen, cx, cy, tw, th = random_case(rng, big)
        q = np.zeros(k)
        if not O.orc_lib().orc_histogram(f.ctypes.data, w, h, ch, cx, cy, tw, th, cen.ctypes.data, k, 1, q.ctypes.data):
            continue
        # perturb the start so mean-shift actually moves
        sx, sy = cx + float(rng.uniform(-3, 3)), cy + float(rng.uniform(-3, 3))
        x, y, st = C.c_double(sx), C.c_double(sy), C.c_int(0)
        O.orc_lib().orc_meanshift_step(f.ctypes.data, w, h, ch, C.byref(x), C.byref(y), tw, th, cen.ctypes.data,
                                       q.ctypes.data, k, 20, 0.5, C.byref(st))
        gx, gy, gs = gpu.meanshift_step(f, w, h, ch, sx, sy, tw, th, cen, q, 20, 0.5)
        assert (gx, gy, gs) == (x.value, y.value, st.value), trial
        tested += 1
    assert tested >= 5


def test_meanshift_known_answers(gpu):
    """tracking_test.cpp:201-243."""
    red, yellow = (255, 0, 0), (255, 255, 0)
    cen = np.array([[255, 0, 0], [255, 255, 0], [0, 0, 0]], np.float64)

    def target(x0, y0):
        f = np.zeros((40, 40, 3), np.uint8)
        f[y0:y0 + 9, x0:x0 + 9] = red
        f[y0 + 2:y0 + 7, x0 + 2:x0 + 7] = yellow
        return f.reshape(-1)

    f0 = target(16, 16)
    q = gpu.histogram(f0, 40, 40, 3, 20, 20, 9, 9, cen)
    x, y, st = gpu.meanshift_step(f0, 40, 40, 3, 20.0, 20.0, 9, 9, cen, q, 40, 0.01)
    assert (x, y, st) == (20.0, 20.0, 0)
    x, y, st = gpu.meanshift_step(target(19, 16), 40, 40, 3, 20.0, 20.0, 9, 9, cen, q, 40, 0.01)
    assert st == 0 and abs(x - 23) <= 1 and abs(y - 20) <= 1
    x, y, st = gpu.meanshift_step(np.zeros(40 * 40 * 3, np.uint8), 40, 40, 3, 20.0, 20.0, 9, 9, cen, q, 40, 0.01)
    assert st == 1
    x, y, st = gpu.meanshift_step(f0, 40, 40, 3, 20.0, 20.0, 9, 9, cen, q, 40, 0.01, status=1)
    assert (x, y, st) == (20.0, 20.0, 1)


def rect_blobs(c, rects_t):
    m = np.zeros((c.height, c.width), np.uint8)
    for (ix, iy, rw, rh) in rects_t:
        m[iy:iy + rh, ix:ix + rw] = 1
    _, blobs, _ = O.cpu_label(m.reshape(-1), c.width, c.height, 1, 4)
    return blobs


@pytest.mark.parametrize("name,clip,cfg", [
    ("two_squares", two_squares_clip, TRACKER_CFG(k_clusters=4, seed=7)),
    ("acceptance6", acceptance6_clip, TRACKER_CFG()),
])
def test_tracker_golden_logs(gpu, name, clip, cfg):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    c = clip()
    frames, rects = O.orc_frames(c)
    trk = gpu.Tracker(cfg)
    for t in range(c.n_frames):
        trk.process(frames[t], c.width, c.height, c.channels, rect_blobs(c, rects[t]))
    log = trk.log()
    assert log.tobytes() == g["log"].tobytes()
    assert trk.frames_processed == c.n_frames


def test_tracker_spawn_ids_and_model(gpu):
    """tracking_test.cpp:279-300: ids 1 and 2, histograms sum to 1; the
    quantizer and target histogram equal the oracle's bit for bit."""
    c = two_squares_clip()
    frames, rects = O.orc_frames(c, 1)
    cfg = TRACKER_CFG(k_clusters=4, seed=7)
    trk = gpu.Tracker(cfg)
    ref = O.CpuTracker(cfg, "orc")
    blobs = rect_blobs(c, rects[0])
    trk.process(frames[0], c.width, c.height, 3, blobs)
    ref.process(frames[0], c.width, c.height, 3, blobs)
    tr = trk.tracks()
    assert [t.track_id for t in tr] == [1, 2]
    for i in range(2):
        cg, qg = trk.track_model(i)
        cr, qr = ref.track_model(i)
        assert cg.tobytes() == cr.tobytes() and qg.tobytes() == qr.tobytes()
        assert abs(qg.sum() - 1.0) < 1e-9
    trk.process(frames[0], c.width, c.height, 3, blobs)
    assert len(trk.tracks()) == 2


def test_tracker_retires_after_five_lost_frames(gpu):
    """tracking_test.cpp:343-372."""
    f0 = np.zeros((24, 24, 3), np.uint8)
    f0[8:15, 8:15] = (255, 0, 0)
    for cy in (8, 14):
        for cx in (8, 14):
            f0[cy, cx] = (0, 0, 255)
    m = np.zeros(24 * 24, np.uint8).reshape(24, 24)
    m[8:15, 8:15] = 1
    _, blobs, _ = O.cpu_label(m.reshape(-1), 24, 24, 1, 4)
    trk = gpu.Tracker(TRACKER_CFG(k_clusters=2, seed=7))
    trk.process(f0.reshape(-1), 24, 24, 3, blobs)
    assert len(trk.tracks()) == 1
    blue = np.zeros((24, 24, 3), np.uint8)
    blue[:, :] = (0, 0, 255)
    empty = np.zeros(0, BLOB_DTYPE)
    for _ in range(4):
        trk.process(blue.reshape(-1), 24, 24, 3, empty)
        tr = trk.tracks()
        assert len(tr) == 1 and tr[0].status == 1
    trk.process(blue.reshape(-1), 24, 24, 3, empty)
    assert trk.tracks() == []


@pytest.mark.parametrize("name,n", [("C1", 200), ("C2", 150)])
def test_tracker_on_recipe_pipeline(gpu, name, n):
    """Device tracker fed the oracle's blobs on the benchmark recipes."""
    clip = recipe(name)
    frames, _ = O.orc_frames(clip, n)
    out, log, _ = O.run_pipeline_cpu(clip, frames, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), "orc")
    trk = gpu.Tracker(TRACKER_CFG())
    for t, m, lab, blobs in out:
        trk.process(frames[t], clip.width, clip.height, 1, blobs)
    assert trk.log().tobytes() == log.tobytes()

"""CPU: the C-ABI library loads and exports every declared symbol; host-side
logic (synthetic recipes, exact-arithmetic replicas) is correct.  No kernel
is launched here."""
import ctypes as C
import math
import os
import re

import numpy as np
import pytest

import paper_1310_3322_b200 as trb
from paper_1310_3322_b200 import api
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import Rng, lround, mix_seed, recipe
from tests import _oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    hdr = open(os.path.join(ROOT, "include", "trb.h")).read()
    return sorted(set(re.findall(r"\b(trb_[a-z0-9_]+)\s*\(", hdr)))


def test_library_exports_every_declared_symbol():
    L = C.CDLL(api.build())
    syms = declared_symbols()
    assert len(syms) > 40
    for s in syms:
        assert hasattr(L, s), f"libtrb.so does not export {s}"


def test_no_device_fails_loudly_without_gpu():
    """Without a GPU the compute entry points must error, never fall back."""
    if trb.device_count() > 0:
        pytest.skip("a GPU is present")
    with pytest.raises(trb.CudaError):
        trb.MotionDetector(MOTION_CFG(window=5), 8, 8)
    with pytest.raises(trb.CudaError):
        trb.label_blocked(np.zeros(64, np.uint8), 8, 8)


def test_argument_errors_before_any_device_work():
    """New entry points reject bad arguments with the C ABI's status codes
    (1 = invalid argument) before touching a device."""
    L = trb.lib()
    L.trb_streams_join.argtypes = [C.c_void_p, C.c_void_p]
    assert L.trb_streams_join(None, None) == 1
    assert b"null argument" in L.trb_last_error()
    L.trb_morph_device.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p]
    buf = C.c_void_p(1)
    assert L.trb_morph_device(None, buf, 16, 16, 1, 3, None) == 1
    assert L.trb_morph_device(buf, buf, 0, 16, 1, 3, None) == 1
    assert b"positive dimensions" in L.trb_last_error()
    assert L.trb_morph_device(buf, buf, 16, 16, 1, 9, None) == 1
    assert b"unknown morphology op" in L.trb_last_error()


def test_config_validation_messages():
    L = trb.lib()
    assert L.trb_motion_config_validate(C.byref(MOTION_CFG(window=1))) == 2
    assert b"window_w" in L.trb_last_error()
    assert L.trb_motion_config_validate(C.byref(MOTION_CFG(threshold=255))) == 2
    assert L.trb_motion_config_validate(C.byref(MOTION_CFG(bins=257))) == 2
    assert L.trb_motion_config_validate(C.byref(MOTION_CFG(method=1, window=2, threshold=254, bins=2))) == 0
    assert L.trb_seg_config_validate(C.byref(SEG_CFG(0, 1, 1))) == 2
    assert L.trb_seg_config_validate(C.byref(SEG_CFG(1, 1, 0))) == 2
    assert L.trb_tracker_config_validate(C.byref(TRACKER_CFG(k_clusters=1))) == 2
    assert L.trb_tracker_config_validate(C.byref(TRACKER_CFG(eps=0.0))) == 2
    assert L.trb_tracker_config_validate(C.byref(TRACKER_CFG(max_iters=0))) == 2
    assert L.trb_tracker_config_validate(C.byref(TRACKER_CFG(kmeans_iters=0))) == 2
    assert L.trb_tracker_config_validate(C.byref(TRACKER_CFG())) == 0


def test_rng_matches_oracle_mt19937_64():
    # std::mt19937_64 reference value: the 10000th output for the default seed
    r = Rng(5489)
    for _ in range(9999):
        r.next_u64()
    assert r.next_u64() == 9981545732273789042
    assert mix_seed(3, 0) == O.orc_lib().orc_mix_seed(3, 0)
    assert mix_seed(1003, 17) == O.orc_lib().orc_mix_seed(1003, 17)


def test_lround_half_away_from_zero():
    assert lround(2.5) == 3 and lround(-2.5) == -3 and lround(0.49999999999999994) == 0
    assert lround(1.4999999999999998) == 1


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4"])
def test_recipes_stay_in_frame_and_match_oracle_raster(name):
    clip = recipe(name)
    rects = clip.all_rects()  # raises if a shape leaves the frame
    assert len(rects) == clip.n_frames
    if name in ("C1", "C2"):
        frames, orects = O.orc_frames(clip, 40)
        assert (np.array(rects[:40], np.int32) == orects).all()
        from paper_1310_3322_b200.synth import raster_host
        for t in (0, 17, 39):
            assert (raster_host(clip, rects[t]) == frames[t]).all()


def test_glibc_hypot_replica_matches_libm_host():
    """trb_exact.cuh's glibc_hypot (host build) == the live libm hypot."""
    rng = np.random.default_rng(1)
    n = 400000
    x = np.concatenate([rng.uniform(-4000, 4000, n), rng.standard_normal(n) * 1e-3,
                        rng.integers(-50, 50, n).astype(np.float64) + rng.choice([0.0, 0.5, 0.25], n),
                        np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-1074, 1023, n))])
    y = np.concatenate([rng.uniform(-4000, 4000, n), rng.standard_normal(n) * 1e-3,
                        rng.integers(-50, 50, n).astype(np.float64),
                        np.ldexp(rng.uniform(0.5, 1, n), rng.integers(-1074, 1023, n))])
    got = api.selftest_hypot(x, y, on_device=False)
    L = O.orc_lib()
    want = np.array([L.orc_libm_hypot(a, b) for a, b in zip(x, y)])
    assert got.tobytes() == want.tobytes()
    assert math.hypot(3.0, 4.0) == 5.0

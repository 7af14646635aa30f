"""Seeded configuration fuzz against the UNMODIFIED reference (oracle/_ref):
odd frame sizes (widths not multiples of 16), gray and RGB clips, Mean and
Mode backgrounds with windows 2..300 (both sum widths, incremental and
re-read Mode), both connectivities, block
grids, min_area, and tracker settings (k_clusters, max_iters, eps,
kmeans_iters, seed).  Every steady frame's mask / label planes, blob table
and the whole track log of every stream must be identical."""
import numpy as np
import pytest

from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import Clip, Shape
from tests import _oracle as O
from tests.test_gpu_bench_parity import compare

pytestmark = pytest.mark.gpu

N_CASES = 40


def make_case(seed):
    rng = np.random.default_rng(seed)
    w = int(rng.integers(64, 360))
    h = int(rng.integers(48, 260))
    ch = int(rng.choice([1, 1, 3]))
    # windows across the kernels' regimes: u16 sums (<= 257) / u32, incremental Mode (<= 255) / ring re-read
    window = int(rng.choice([2, 5, 17, 40, 91, 255, 256, 300]))
    steady = 25
    n = window - 1 + steady
    clips = []
    for s in range(2):
        shapes = []
        for _ in range(int(rng.integers(1, 6))):
            sw, sh = int(rng.integers(6, min(32, w // 3))), int(rng.integers(6, min(32, h // 3)))
            col = tuple(int(c) for c in (rng.integers(60, 256, 3) if ch == 3 else [rng.integers(60, 256)] * 3))
            x0 = float(rng.uniform(0, w - sw - 1))
            y0 = float(rng.uniform(0, h - sh - 1))
            x1 = float(rng.uniform(0, w - sw - 1))
            y1 = float(rng.uniform(0, h - sh - 1))
            span = max(1, n - 1)
            shapes.append(Shape(sw, sh, col, x0, y0, (x1 - x0) / span, (y1 - y0) / span))
        clips.append(Clip(w, h, ch, int(rng.integers(0, 40)), shapes, n, int(rng.integers(1, 1 << 30)), f"fuzz{seed}.{s}"))
    method = int(rng.integers(0, 2))
    mcfg = MOTION_CFG(method=method, window=window, threshold=int(rng.choice([5, 25, 60])),
                      bins=int(rng.choice([8, 16, 32, 64])))
    scfg = SEG_CFG(n_blocks=int(rng.choice([1, 2, 4, 7])), connectivity=int(rng.integers(0, 2)),
                   min_area=int(rng.choice([1, 4, 15])))
    tcfg = TRACKER_CFG(k_clusters=int(rng.choice([2, 4, 8, 16, 24])),  # 24: past the v2 engine's lanes max_iters=int(rng.choice([1, 3, 20])),
                       eps=float(rng.choice([0.1, 0.5, 3.0])), kmeans_iters=int(rng.choice([1, 5, 20])),
                       seed=int(rng.integers(0, 1 << 62)))
    return clips, n, mcfg, scfg, tcfg


def run_device(trb, clips, frames, n, mcfg, scfg, tcfg):
    import torch
    c0 = clips[0]
    S = len(clips)
    dev = [torch.from_numpy(f).cuda() for f in frames]
    st = trb.Streams(S, c0.width, c0.height, c0.channels, mcfg, scfg, tcfg)
    per = [dict(hashes=[], nblobs=[], blobs=[]) for _ in range(S)]
    for t in range(n):
        st.step_device([dev[s][t].data_ptr() for s in range(S)])
        if not st.has_output:
            continue
        for s in range(S):
            per[s]["hashes"].append((O.plane_hash(st.mask(s)), O.plane_hash(st.labels(s))))
            b = st.blobs(s)
            per[s]["nblobs"].append(len(b))
            per[s]["blobs"].append(b)
    st.synchronize()
    for s in range(S):
        per[s]["hashes"] = np.array(per[s]["hashes"], np.uint64).reshape(-1, 2)
        per[s]["log"] = st.log(s)
    return per


@pytest.mark.parametrize("seed", range(N_CASES))
def test_config_fuzz_vs_reference(gpu, seed):
    if not O.ref_available():
        pytest.fail("oracle/_ref/libteamrec_ref.so missing: build it with make -C oracle where the reference is")
    clips, n, mcfg, scfg, tcfg = make_case(seed)
    frames = [O.ref_frames(c, n)[0] for c in clips]
    c0 = clips[0]
    ref = O.ref_run_streams_detail(frames, c0.width, c0.height, c0.channels, mcfg, scfg, tcfg, 2, bcap=64,
                                   lcap=16384)
    got = run_device(gpu, clips, frames, n, mcfg, scfg, tcfg)
    compare(got, ref)
    assert all(len(g["hashes"]) == n - mcfg.window + 1 for g in got)


def make_case_1080p(seed):
    """Full-HD clips (the v1 mean-shift engine, 8-16-CTA clusters) under
    non-default configurations."""
    from paper_1310_3322_b200.synth import random_clip
    rng = np.random.default_rng(1000 + seed)
    window = int(rng.choice([17, 40, 91]))
    n = window - 1 + 15
    clips = [random_clip(1920, 1080, int(rng.integers(6, 20)), 30, 90, bool(rng.integers(0, 2)),
                         int(rng.integers(1, 1 << 30)), int(rng.integers(1, 1 << 30)), n) for _ in range(2)]
    mcfg = MOTION_CFG(method=int(rng.integers(0, 2)), window=window, threshold=int(rng.choice([10, 25, 40])),
                      bins=int(rng.choice([16, 32])))
    scfg = SEG_CFG(n_blocks=int(rng.choice([1, 4, 9])), connectivity=int(rng.integers(0, 2)),
                   min_area=int(rng.choice([1, 4, 30])))
    tcfg = TRACKER_CFG(k_clusters=int(rng.choice([4, 8, 16, 24])), max_iters=int(rng.choice([5, 20])),
                       eps=float(rng.choice([0.25, 0.5, 1.0])), kmeans_iters=int(rng.choice([5, 20])),
                       seed=int(rng.integers(0, 1 << 62)))
    return clips, n, mcfg, scfg, tcfg


@pytest.mark.parametrize("seed", range(8))
def test_config_fuzz_1080p_vs_reference(gpu, seed):
    if not O.ref_available():
        pytest.fail("oracle/_ref/libteamrec_ref.so missing: build it with make -C oracle where the reference is")
    clips, n, mcfg, scfg, tcfg = make_case_1080p(seed)
    frames = [O.ref_frames(c, n)[0] for c in clips]
    ref = O.ref_run_streams_detail(frames, 1920, 1080, 1, mcfg, scfg, tcfg, 2, bcap=64, lcap=16384)
    got = run_device(gpu, clips, frames, n, mcfg, scfg, tcfg)
    compare(got, ref)
    assert sum(len(g["log"]) for g in got) > 0

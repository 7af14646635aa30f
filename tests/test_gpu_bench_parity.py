"""GPU parity on the benchmark's own work, against the UNMODIFIED reference
(oracle/_ref: the reference headers compiled behind a C shim), not the C
restatement:

* the device-rasterised bench frames are the reference generator's frames
  (synth_frames, synth.hpp:45-101), every stream and every frame the bench
  touches;
* all 64 C5 streams through frame 134 (the bench's 90 fill + warm-up +
  timed + profile frames) — per steady frame the mask and label planes
  (plane_hash digests), the blob tables, and the whole track log;
* the full 300-frame C3 clip (BASELINE configs[2]), 8 C5 streams through
  the whole 300-frame clip, and 60 steady C4 frames (configs[3]) the same way;
* the glibc hypot replica that decides gating and convergence on 1e8 device
  samples.
Steps run exactly as bench.py issues them (step_device on device frames,
step overlap on); outputs are read back between steps.
"""
import numpy as np
import pytest

from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import device_frames, recipe
from tests import _oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

BENCH_FRAMES = 135  # bench.py default: 90 fill + 5 warm-up + 20 timed + 20 profile steps


def _need_ref():
    if not O.ref_available():
        pytest.fail("oracle/_ref/libteamrec_ref.so missing: build it with make -C oracle where the reference is")


def run_gpu(trb, clips, n_frames, torch_stream=None):
    """The bench's sequence (step_device over device frames, overlap on),
    reading every steady step's planes back.  Per stream: hashes [k, 2]
    (mask, labels), nblobs [k], blobs (list of arrays), log."""
    import torch
    c0 = clips[0]
    S = len(clips)
    stream = torch.cuda.Stream()
    frames = device_frames(clips, n_frames, stream.cuda_stream)
    st = trb.Streams(S, c0.width, c0.height, c0.channels, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    per = [dict(hashes=[], nblobs=[], blobs=[]) for _ in range(S)]
    with torch.cuda.stream(stream):
        for t in range(n_frames):
            st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
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
    del frames
    return per


def compare(per_gpu, per_ref, bcap=64):
    for s, (g, r) in enumerate(zip(per_gpu, per_ref)):
        assert len(g["hashes"]) == len(r["hashes"]), f"stream {s}: steady frame count"
        bad = np.nonzero((g["hashes"] != r["hashes"]).any(axis=1))[0]
        assert bad.size == 0, f"stream {s}: mask/label planes differ at steady frames {bad[:8]}"
        assert (np.array(g["nblobs"]) == r["nblobs"]).all(), f"stream {s}: blob counts"
        for k, b in enumerate(g["blobs"]):
            n = min(len(b), bcap)
            assert b[:n].tobytes() == r["blobs"][k, :n].tobytes(), f"stream {s} steady frame {k}: blob table"
        assert g["log"].tobytes() == r["log"].tobytes(), f"stream {s}: track log"


def ref_batches(clips, n_frames, batch=16, threads=16):
    """The reference loop over the reference generator's own frames, streams
    in batches (the frames of a batch are held in host memory)."""
    out = []
    c0 = clips[0]
    for b0 in range(0, len(clips), batch):
        fr = [O.ref_frames(c, n_frames)[0] for c in clips[b0:b0 + batch]]
        out += O.ref_run_streams_detail(fr, c0.width, c0.height, c0.channels, MOTION_CFG(), SEG_CFG(),
                                        TRACKER_CFG(), threads, bcap=64, lcap=8192)
        del fr
    return out


def test_bench_device_frames_are_reference_synth_frames(gpu):
    """Every frame the bench touches (64 C5 streams x frames 0..134) hashes
    equal to the reference generator's frame (synth_frames)."""
    _need_ref()
    import torch
    clips = [recipe("C5", s) for s in range(64)]
    for b0 in range(0, 64, 8):
        dev = device_frames(clips[b0:b0 + 8], BENCH_FRAMES).cpu().numpy()
        for i, c in enumerate(clips[b0:b0 + 8]):
            ref, _ = O.ref_frames(c, BENCH_FRAMES)
            for t in range(BENCH_FRAMES):
                assert O.plane_hash(dev[i, t]) == O.plane_hash(ref[t]), f"stream {b0 + i} frame {t}"
            assert dev[i].tobytes() == ref.tobytes()
        del dev
        torch.cuda.empty_cache()


def test_c5_all_64_streams_through_bench_frames_vs_reference(gpu):
    """All 64 C5 streams through frame 134 (45 steady frames each) against
    the unmodified reference: planes, blob tables, whole track logs."""
    _need_ref()
    clips = [recipe("C5", s) for s in range(64)]
    per_gpu = run_gpu(gpu, clips, BENCH_FRAMES)
    per_ref = ref_batches(clips, BENCH_FRAMES)
    compare(per_gpu, per_ref)
    assert sum(len(g["log"]) for g in per_gpu) > 64 * 45  # tracks were live throughout


def test_c5_streams_full_300_frame_clips_vs_reference(gpu):
    """Past the bench's frames: 8 C5 streams (stream seeds 60..67: four of the
    bench's and four beyond) through the whole 300-frame clip — every steady frame's planes and
    blob table and the whole track log, as the e2e leg's later frames see."""
    _need_ref()
    clips = [recipe("C5", s) for s in range(60, 68)]
    per_gpu = run_gpu(gpu, clips, 300)
    per_ref = ref_batches(clips, 300, batch=8, threads=8)
    compare(per_gpu, per_ref)
    assert all(len(g["hashes"]) == 210 for g in per_gpu)


def test_c3_full_300_frame_clip_vs_reference(gpu):
    """BASELINE configs[2]: the 300-frame 1080p clip (shape seed 3, 20 blobs
    with occlusions/merges), full label + blob-stat + track output."""
    _need_ref()
    clip = recipe("C3")
    per_gpu = run_gpu(gpu, [clip], 300)
    per_ref = ref_batches([clip], 300, threads=1)
    compare(per_gpu, per_ref)
    assert len(per_gpu[0]["hashes"]) == 210


def test_c4_60_steady_frames_vs_reference(gpu):
    """BASELINE configs[3]: 3840x2160, 50 blobs (CCL seam-merge stress),
    the window fill plus 60 steady frames."""
    _need_ref()
    clip = recipe("C4")
    per_gpu = run_gpu(gpu, [clip], 150)
    per_ref = ref_batches([clip], 150, threads=1)
    compare(per_gpu, per_ref)
    assert len(per_gpu[0]["hashes"]) == 60


def test_glibc_hypot_1e8_device_samples(gpu):
    """trb_exact.cuh's glibc_hypot on the device == the live libm hypot on
    1e8 inputs: centroid shifts and gating distances (|d| up to a frame,
    quarter/half-pixel fractions, tiny shifts near eps) plus random
    binades over the whole double range."""
    from paper_1310_3322_b200 import api
    rng = np.random.default_rng(20261019)
    n_chunk, total = 10_000_000, 0
    for chunk in range(10):
        k = n_chunk // 5
        x = np.concatenate([rng.uniform(-4000, 4000, k), rng.standard_normal(k) * 0.5,
                            rng.integers(-3840, 3840, k) + rng.choice([0.0, 0.25, 0.5, 0.75], k),
                            rng.uniform(-1, 1, k) * np.ldexp(1.0, rng.integers(-60, 12, k)),
                            np.ldexp(rng.uniform(0.5, 1, k), rng.integers(-1074, 1023, k)) * rng.choice([-1, 1], k)])
        y = np.concatenate([rng.uniform(-4000, 4000, k), rng.standard_normal(k) * 0.5,
                            rng.integers(-2160, 2160, k) + rng.choice([0.0, 0.5], k),
                            rng.uniform(-1, 1, k) * np.ldexp(1.0, rng.integers(-60, 12, k)),
                            np.ldexp(rng.uniform(0.5, 1, k), rng.integers(-1074, 1023, k)) * rng.choice([-1, 1], k)])
        got = api.selftest_hypot(x, y, on_device=True)
        want = O.libm_hypot(x, y)
        assert got.tobytes() == want.tobytes(), f"chunk {chunk}"
        total += x.size
    assert total == 100_000_000

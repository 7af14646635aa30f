"""GPU parity of the batched, device-resident front end (the bench path):
several streams advance together, masks / labels / blobs / track logs of
every stream are bit-identical to the reference pipeline (golden fixtures)
and to the oracle."""
import os

import numpy as np
import pytest

from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import bench_vision_clip, harness_vision_clip, recipe
from tests import _oracle as O
from tests.golden.make_golden import sha

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def run_streams(trb, clips, n, mcfg, host=True):
    c0 = clips[0]
    frames = [O.orc_frames(c, n)[0] for c in clips]
    st = trb.Streams(len(clips), c0.width, c0.height, c0.channels, mcfg, SEG_CFG(), TRACKER_CFG())
    per = [dict(mask_sha=[], label_sha=[], nblobs=[], blobs=[]) for _ in clips]
    import torch
    dev = [torch.from_numpy(f).cuda() for f in frames] if not host else None
    for t in range(n):
        if host:
            st.step_host([frames[s][t] for s in range(len(clips))])
        else:
            st.step_device([dev[s][t].data_ptr() for s in range(len(clips))])
        if st.has_output:
            for s in range(len(clips)):
                per[s]["mask_sha"].append(sha(st.mask(s)))
                per[s]["label_sha"].append(sha(st.labels(s)))
                b = st.blobs(s)
                per[s]["nblobs"].append(len(b))
                per[s]["blobs"].append(b)
    st.synchronize()
    for s in range(len(clips)):
        per[s]["log"] = st.log(s)
        per[s]["blobs"] = np.concatenate(per[s]["blobs"]) if per[s]["blobs"] else None
    return per


@pytest.mark.parametrize("name,clip,n,window", [
    ("c1_pipeline", lambda: recipe("C1"), 160, 91),
    ("harness_vision", harness_vision_clip, 29, 9),
    ("bench_vision", bench_vision_clip, 151, 91),
    ("c2_pipeline", lambda: recipe("C2"), 140, 91),
])
def test_streams_match_reference_golden(gpu, name, clip, n, window):
    g = np.load(os.path.join(GOLD, name + ".npz"))
    per = run_streams(gpu, [clip(), clip()], n, MOTION_CFG(window=window))
    for s in range(2):
        r = per[s]
        assert (np.array(r["mask_sha"]) == g["mask_sha"]).all()
        assert (np.array(r["label_sha"]) == g["label_sha"]).all()
        assert (np.array(r["nblobs"]) == g["nblobs"]).all()
        assert r["blobs"].tobytes() == g["blobs"].tobytes()
        assert r["log"].tobytes() == g["log"].tobytes()


def test_streams_distinct_c5_streams_device_inputs(gpu):
    """Three different C5 streams (1080p) from device-resident inputs vs
    the oracle pipeline, 100 frames each (10 steady)."""
    clips = [recipe("C5", s) for s in range(3)]
    n = 100
    per = run_streams(gpu, clips, n, MOTION_CFG(), host=False)
    for s, c in enumerate(clips):
        frames, _ = O.orc_frames(c, n)
        out, log, _ = O.run_pipeline_cpu(c, frames, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), "orc")
        assert per[s]["mask_sha"] == [sha(m) for _, m, _, _ in out]
        assert per[s]["label_sha"] == [sha(l_) for _, _, l_, _ in out]
        assert per[s]["log"].tobytes() == log.tobytes()


@pytest.mark.parametrize("pinned", [True, False, "contiguous"])
def test_streams_pipelined_host_steps_match_golden(gpu, pinned):
    """step_host_async (H2D on the copy stream into double-buffered staging,
    overlapping the previous step; results land asynchronously): per-step
    blob counts and the final track logs equal the reference's."""
    import torch
    name, clip, n, window = "c1_pipeline", recipe("C1"), 160, 91
    g = np.load(os.path.join(GOLD, name + ".npz"))
    frames = O.orc_frames(clip, n)[0]
    if pinned == "contiguous":  # both streams' frames back to back: one coalesced H2D copy per step
        pairs = [torch.from_numpy(np.stack([frames[t], frames[t]])).pin_memory().numpy() for t in range(n)]
        res = torch.zeros((n, 2), dtype=torch.int32).pin_memory().numpy()
    elif pinned:
        host = [torch.from_numpy(frames[t]).pin_memory().numpy() for t in range(n)]
        pairs = [[host[t], host[t]] for t in range(n)]
        res = torch.zeros((n, 2), dtype=torch.int32).pin_memory().numpy()
    else:
        host = [frames[t].copy() for t in range(n)]
        pairs = [[host[t], host[t]] for t in range(n)]
        res = np.zeros((n, 2), np.int32)
    st = gpu.Streams(2, clip.width, clip.height, clip.channels, MOTION_CFG(window=window), SEG_CFG(), TRACKER_CFG())
    for t in range(n):
        st.step_host_async([pairs[t][0], pairs[t][1]], res[t])
    st.synchronize()
    emitted = res[window - 1:]
    for s in range(2):
        assert (emitted[:, s] == g["nblobs"]).all()
        assert st.log(s).tobytes() == g["log"].tobytes()
    assert (res[:window - 1] == 0).all()


def test_streams_blob_features_vs_oracle(gpu):
    """extract_blob_features on a stream's device labels / blobs and its
    frame in HBM (trb_streams_blob_features) vs the oracle on the same step."""
    import torch
    clips = [recipe("C1"), recipe("C1")]
    n = 100
    frames = [O.orc_frames(c, n)[0] for c in clips]
    dev = [torch.from_numpy(f).cuda() for f in frames]
    c0 = clips[0]
    st = gpu.Streams(2, c0.width, c0.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    for t in range(n):
        st.step_device([dev[s][t].data_ptr() for s in range(2)])
    st.synchronize()
    for s in range(2):
        mean, aspect = st.blob_features(s, dev[s][n - 1].data_ptr())
        labels, blobs = st.labels(s), st.blobs(s)
        om, oa = O.cpu_blob_features(labels, c0.width, c0.height, frames[s][n - 1], c0.width, c0.height, 1, blobs)
        assert len(mean) == len(blobs) > 0
        assert mean.tobytes() == om.tobytes() and aspect.tobytes() == oa.tobytes()


def test_streams_warp_matches_reference_stream_detect(gpu):
    """MotionConfig(warp=homography): frames warped into the reference plane
    on the device before the window (stream_detect, motion.hpp:260-282); the
    masks equal the reference's stream_detect output (golden)."""
    import torch
    from paper_1310_3322_b200.api import InvalidArgument
    g = np.load(os.path.join(GOLD, "warp.npz"))
    clip = harness_vision_clip()
    frames, homs = g["stream_frames"], g["stream_homs"]
    mcfg = MOTION_CFG(window=9)
    mcfg.warp = 1
    dev = torch.from_numpy(frames).cuda()
    st = gpu.Streams(2, clip.width, clip.height, clip.channels, mcfg, SEG_CFG(), TRACKER_CFG())
    with pytest.raises(InvalidArgument, match="requires per-frame homographies"):
        st.step_device([dev[0].data_ptr()] * 2)
    masks = []
    for t in range(frames.shape[0]):
        st.step_device_warp([dev[t].data_ptr()] * 2, np.stack([homs[t], homs[t]]))
        if st.has_output:
            masks.append((st.mask(0).copy(), st.mask(1).copy()))
    st.synchronize()
    assert len(masks) == len(g["stream_masks"])
    for (m0, m1), ref in zip(masks, g["stream_masks"]):
        assert m0.tobytes() == ref.tobytes() and m1.tobytes() == ref.tobytes()


def test_streams_overlapped_steps_without_sync(gpu):
    """The bench's issue pattern: device-resident C5 steps enqueued back to
    back on a user stream with no host sync (each step's tracking overlaps
    the next step's motion + CCL on the internal stream; blob tables
    double-buffered), then join(): track logs equal the oracle's and the
    in-stream (TRB_OVERLAP=0) run's."""
    import torch
    clips = [recipe("C5", s) for s in (5, 6)]
    n = 100
    frames = [O.orc_frames(c, n)[0] for c in clips]
    dev = [torch.from_numpy(f).cuda() for f in frames]
    logs = {}
    for ov in ("1", "0"):
        os.environ["TRB_OVERLAP"] = ov
        try:
            st = gpu.Streams(2, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
        finally:
            os.environ.pop("TRB_OVERLAP")
        stream = torch.cuda.Stream()
        for t in range(n):
            st.step_device([dev[s][t].data_ptr() for s in range(2)], stream.cuda_stream)
        st.join(stream.cuda_stream)
        stream.synchronize()  # the join alone must cover the last step's tracking
        logs[ov] = [st.log(s).tobytes() for s in range(2)]
        st.synchronize()
    assert logs["1"] == logs["0"]
    out, log, _ = O.run_pipeline_cpu(clips[0], frames[0], MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), "orc")
    assert logs["1"][0] == log.tobytes()


def test_streams_overlap_profiling_switches(gpu):
    """Switching a handle between the overlapped path and the in-stream
    (per-stage profiling) path every few steps, device and host-async steps
    mixed, no host sync between steps: the track log still equals the
    oracle's (the switch joins the tracker stream before in-stream tracking)."""
    import torch
    clip = recipe("C5", 7)
    n = 100
    frames = O.orc_frames(clip, n)[0]
    dev = torch.from_numpy(frames).cuda()
    host = [torch.from_numpy(frames[t]).pin_memory().numpy() for t in range(n)]
    st = gpu.Streams(1, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    stream = torch.cuda.Stream()
    for t in range(n):
        st.profile((t // 3) % 2 == 1)
        if t % 5 == 4:
            st.step_host_async([host[t]], None, stream.cuda_stream)
        else:
            st.step_device([dev[t].data_ptr()], stream.cuda_stream)
    st.profile(False)
    st.synchronize()
    _, log, _ = O.run_pipeline_cpu(clip, frames, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), "orc")
    assert st.log(0).tobytes() == log.tobytes()


def test_streams_c4_4k_end_to_end(gpu):
    """BASELINE configs[3] (3840x2160, 50 blobs, crossing paths): masks,
    labels and the track log of the batched device path vs the oracle over
    the window fill and 7 steady frames."""
    import torch
    clip = recipe("C4")
    n = 98
    frames = O.orc_frames(clip, n)[0]
    dev = torch.from_numpy(frames).cuda()
    st = gpu.Streams(1, clip.width, clip.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    masks, labels = [], []
    for t in range(n):
        st.step_device([dev[t].data_ptr()])
        if st.has_output:
            masks.append(sha(st.mask(0)))
            labels.append(sha(st.labels(0)))
    st.synchronize()
    out, log, _ = O.run_pipeline_cpu(clip, frames, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), "orc")
    assert masks == [sha(m) for _, m, _, _ in out]
    assert labels == [sha(l_) for _, _, l_, _ in out]
    assert len(log) > 0 and st.log(0).tobytes() == log.tobytes()

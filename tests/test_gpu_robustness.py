"""Production robustness of the streams handle: the drainable track-log
ring, the configurable track capacity (overflow fails the step instead of
diverging from the reference), misaligned device frames, and the per-step
result readback (trb_step_output) against the downloaded state."""
from types import SimpleNamespace

import numpy as np
import pytest

from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import random_clip, recipe
from tests import _oracle as O

pytestmark = pytest.mark.gpu


def many_tracks_clip(n_frames):
    """128x96, 24 small non-crossing shapes: ~24 live tracks every frame."""
    return random_clip(128, 96, 24, 5, 7, False, 77, 1077, n_frames, name="many")


def test_log_ring_70k_entries_drained(gpu):
    """A 3000-frame run logging > 70k entries through a 65,536-entry ring:
    drained every 500 steps, the concatenated log equals the oracle's; the
    same run without draining fails with CapacityError when the ring fills."""
    n = 3000
    clip = many_tracks_clip(n)
    frames, _ = O.orc_frames(clip, n)
    mcfg = MOTION_CFG(window=2)
    _, want, _ = O.run_pipeline_cpu(clip, frames, mcfg, SEG_CFG(), TRACKER_CFG(), "orc")
    assert len(want) > 70_000
    st = gpu.Streams(1, clip.width, clip.height, 1, mcfg, SEG_CFG(), TRACKER_CFG())
    parts = []
    for t in range(n):
        st.step_host([frames[t]])
        if t % 500 == 499:
            parts.append(st.drain_log(0))
    st.synchronize()
    parts.append(st.drain_log(0))
    got = np.concatenate(parts)
    assert got.tobytes() == want.tobytes()
    assert len(st.log(0)) == 0  # everything drained

    st2 = gpu.Streams(1, clip.width, clip.height, 1, mcfg, SEG_CFG(), TRACKER_CFG())
    with pytest.raises(gpu.api.CapacityError, match="track-log ring full"):
        for t in range(n):
            st2.step_host([frames[t]])
        st2.synchronize()
    # the entries the ring held before the failing step are intact
    held = st2.log(0)
    assert len(held) <= 1 << 16
    assert held.tobytes() == want[:len(held)].tobytes()


def burst_frames(n_blobs=300):
    """640x480 gray: frame 0 background, then a grid of n_blobs 4x4 squares
    20 px apart (outside each other's 1.5 x diagonal gates)."""
    w, h = 640, 480
    f0 = np.full((h, w), 16, np.uint8)
    f1 = f0.copy()
    k = 0
    for y in range(10, h - 10, 20):
        for x in range(10, w - 10, 20):
            if k < n_blobs:
                f1[y:y + 4, x:x + 4] = 200
                k += 1
    assert k == n_blobs
    return SimpleNamespace(width=w, height=h, channels=1), [f0.reshape(-1), f1.reshape(-1), f1.reshape(-1).copy()]


def test_track_capacity_burst(gpu):
    """300 spawns in one frame: the default 256-track capacity fails the step
    (CapacityError, not a silently different tracker); track_cap=512
    reproduces the oracle exactly."""
    clip, frames = burst_frames(300)
    mcfg = MOTION_CFG(window=2)
    _, want, _ = O.run_pipeline_cpu(clip, frames, mcfg, SEG_CFG(), TRACKER_CFG(), "orc")
    assert len({int(e["track_id"]) for e in want}) >= 257
    st = gpu.Streams(1, clip.width, clip.height, 1, mcfg, SEG_CFG(), TRACKER_CFG())
    with pytest.raises(gpu.api.CapacityError, match="track capacity"):
        for f in frames:
            st.step_host([f])
        st.synchronize()
    with pytest.raises(gpu.api.CapacityError):  # sticky: the handle stays failed
        st.step_host([frames[-1]])
    big = gpu.Streams(1, clip.width, clip.height, 1, mcfg, SEG_CFG(), TRACKER_CFG(), track_cap=512)
    for f in frames:
        big.step_host([f])
    big.synchronize()
    assert big.log(0).tobytes() == want.tobytes()


def test_misaligned_device_frames(gpu):
    """Frames at odd byte offsets (a tensor view) take the scalar path:
    same masks / labels / logs as 16-byte aligned frames, no fault."""
    import torch
    clip = recipe("C1")
    n = 100
    frames, _ = O.orc_frames(clip, n)
    px = clip.width * clip.height
    raw = torch.zeros(n * px + 64, dtype=torch.uint8, device="cuda")
    view = raw[3:3 + n * px].view(n, px)
    view.copy_(torch.from_numpy(frames).cuda())
    al = torch.from_numpy(frames).cuda()
    a = gpu.Streams(1, clip.width, clip.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    b = gpu.Streams(1, clip.width, clip.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    for t in range(n):
        assert view[t].data_ptr() % 16 == 3
        a.step_device([al[t].data_ptr()])
        b.step_device([view[t].data_ptr()])
        if a.has_output:
            assert a.mask(0).tobytes() == b.mask(0).tobytes()
            assert a.labels(0).tobytes() == b.labels(0).tobytes()
    a.synchronize()
    b.synchronize()
    assert a.log(0).tobytes() == b.log(0).tobytes() and len(a.log(0)) > 0


def test_step_output_matches_downloads(gpu):
    """trb_streams_step_host_async_out: per step the blob tables and the
    log entries the frame appended, equal to the oracle's per-frame blobs
    and log; frames without a mask report zero counts."""
    import torch
    clip = recipe("C1")
    n = 140
    frames = O.orc_frames(clip, n)[0]
    out, want_log, _ = O.run_pipeline_cpu(clip, frames, MOTION_CFG(), SEG_CFG(), TRACKER_CFG(), "orc")
    host = [torch.from_numpy(frames[t]).pin_memory().numpy() for t in range(n)]
    st = gpu.Streams(2, clip.width, clip.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    outs = [gpu.api.StepOutput(2, blob_cap=16, log_cap=8) for _ in range(n)]
    for t in range(n):
        st.step_host_async([host[t], host[t]], outs[t])
    st.synchronize()
    by_t = {t: blobs for t, _, _, blobs in out}
    logs = [[], []]
    for t in range(n):
        o = outs[t]
        for s in range(2):
            if t not in by_t:
                assert o.n_blobs[s] == 0 and o.n_log[s] == 0
                continue
            want = by_t[t]
            assert o.n_blobs[s] == len(want)
            assert o.stream_blobs(s).tobytes() == want[:16].tobytes()
            logs[s].append(o.stream_log(s))
    for s in range(2):
        assert np.concatenate(logs[s]).tobytes() == want_log.tobytes()


def test_two_rank_shards_cover_the_job(gpu):
    """bench.py's sharding on the product: two handles (one per "rank" of a
    world of 2, strong split of 4 C5 streams) produce exactly the logs and
    blob tables of one handle over all 4 streams."""
    import bench
    import torch
    from paper_1310_3322_b200.synth import device_frames
    clips = [recipe("C5", s) for s in range(4)]
    n = 100
    frames = device_frames(clips, n)
    c0 = clips[0]

    def run(streams):
        st = gpu.Streams(len(streams), c0.width, c0.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
        for t in range(n):
            st.step_device([frames[s, t].data_ptr() for s in streams])
        st.synchronize()
        return {s: (st.log(i).tobytes(), st.blobs(i).tobytes()) for i, s in enumerate(streams)}

    whole = run(list(range(4)))
    parts = {}
    for r in range(2):
        mine = bench.shard(r, 2, 0, 4)
        assert len(mine) == 2
        parts.update(run(mine))
    assert parts == whole
    del frames
    torch.cuda.empty_cache()

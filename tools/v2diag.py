"""v2 engine diagnostics: standalone histograms / mean-shift steps on C5-like
windows vs the oracle, with the engine's debug counters (fallbacks and their
reasons)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.synth import recipe  # noqa: E402
from tests import _oracle as O  # noqa: E402

clip = recipe("C5", 0)
frames, rects = O.orc_frames(clip, 120)
f = frames[110]
W, H = clip.width, clip.height
rng = np.random.default_rng(5)
api.debug_stats(reset=True)
bad = 0
for trial, (ix, iy, w, h) in enumerate(rects[110][:12]):
    k = 16
    vals = np.unique(f.reshape(H, W)[iy:iy + h, ix:ix + w])
    cen = np.repeat(rng.choice(np.concatenate([vals, [16, 200]]), k).astype(np.float64), 3) + rng.random(3 * k)
    for scale in (1, 3, 6):
        tw, th = w * scale, h * scale
        cx, cy = ix + w / 2 + rng.uniform(-3, 3), iy + h / 2 + rng.uniform(-3, 3)
        want = np.zeros(k)
        ok = O.orc_lib().orc_histogram(f.ctypes.data, W, H, 1, cx, cy, tw, th, cen.ctypes.data, k, 1, want.ctypes.data)
        if not ok:
            continue
        got = trb.histogram(f, W, H, 1, cx, cy, tw, th, cen)
        same = got.tobytes() == want.tobytes()
        bad += not same
        if not same:
            print("MISMATCH", trial, scale, tw * th, np.nonzero(got != want)[0][:8])
print("histograms: bad", bad)
print(api.debug_stats(reset=True))

# the bench workload: 64 C5 streams, device frames, a few steady steps
import torch  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import device_frames  # noqa: E402
S = int(os.environ.get("DIAG_STREAMS", "64"))
clips = [recipe("C5", s) for s in range(S)]
fr = device_frames(clips, 100)
st = trb.Streams(S, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
for t in range(100):
    if t == 95:
        api.debug_stats(reset=True)
    st.step_device([fr[s, t].data_ptr() for s in range(S)])
st.synchronize()
print("C5 steps 95-99:", api.debug_stats(reset=True))

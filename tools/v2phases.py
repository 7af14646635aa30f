"""Per-phase time of the v2 exact-sum engine (diagnostics build): mean
microseconds per mean-shift iteration by window-size bucket, seen by thread
0 of the group's rank-0 CTA.  Usage: TRB_ENGINE=2 python tools/v2phases.py [streams]"""
import os
import sys

_DIAG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1310_3322_b200",
                     "libtrb_diag.so")
os.environ.setdefault("TRB_LIB", _DIAG)
os.environ.setdefault("TRB_ENGINE", "2")

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import device_frames, recipe  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
cfg = sys.argv[2] if len(sys.argv) > 2 else "C5"
steps = 5
clips = [recipe("C5", s) for s in range(S)] if cfg == "C5" else [recipe(cfg)] * S
n = 95 + steps
frames = device_frames(clips, n)
st = trb.Streams(S, clips[0].width, clips[0].height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
for t in range(95):
    st.step_device([frames[s, t].data_ptr() for s in range(S)])
st.synchronize()
api.debug_itlog(True)
for t in range(95, n):
    st.step_device([frames[s, t].data_ptr() for s in range(S)])
st.synchronize()
ph = api.debug_phases().astype(float)
api.debug_itlog(False)
names = {1: "hist A walk", 2: "hist A scan+barrier+carry", 3: "hist B walk", 4: "hist C scan+rank",
         5: "hist C barrier", 6: "hist C pull", 7: "hist C replay",
         8: "bhatt/wsq (+fill/next iter)", 9: "cent A walk", 10: "cent A scan+barrier+carry", 11: "cent B walk",
         12: "cent C scan+rank", 13: "cent C barrier", 14: "cent C pull", 15: "cent C replay", 16: "div/hypot"}
mhz = 1965.0
print("buckets: <5k, 5k-50k, 50k-150k, >150k px; iterations/step:",
      " ".join(f"{ph[b, 0] / steps:8.1f}" for b in range(4)))
tot = np.zeros(4)
for k in sorted(names):
    row = [ph[b, k] / max(1, ph[b, 0]) / mhz for b in range(4)]
    tot += row
    print(f"{k:3d} {names[k]:28s}" + "".join(f"{v:10.2f}" for v in row))
print(f"    {'total us/iteration':28s}" + "".join(f"{v:10.2f}" for v in tot))
print("cluster-us per step:", float(sum(ph[b, 0] * tot[b] for b in range(4)) / steps))
print(api.debug_stats())

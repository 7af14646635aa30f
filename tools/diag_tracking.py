"""Diagnostics: per-step timings and device tracker counters on C5 streams.

python tools/diag_tracking.py --streams 8 --steps 10
"""
import argparse
import os
import sys

# the diagnostics build of the library (make -C paper_1310_3322_b200/csrc diag)
_DIAG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1310_3322_b200",
                     "libtrb_diag.so")
if os.path.exists(_DIAG):
    os.environ.setdefault("TRB_LIB", _DIAG)
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_1310_3322_b200.synth import device_frames  # noqa: E402
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import recipe  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--streams", type=int, default=8)
p.add_argument("--steps", type=int, default=10)
p.add_argument("--start", type=int, default=0, help="extra steady steps before measuring")
p.add_argument("--watch", action="store_true", help="hang watchdog with progress records (slow)")
args = p.parse_args()
S = args.streams
stream = torch.cuda.Stream()
clips = [recipe("C5", s) for s in range(S)]
n = 90 + 3 + args.start + args.steps
frames = device_frames(clips, n, stream.cuda_stream)
st = trb.Streams(S, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
ptrs = [[frames[s, t].data_ptr() for s in range(S)] for t in range(n)]
t = 0
prog = api.debug_progress(4096) if args.watch else None
import threading
state = {"step": -1000, "t": time.time()}


def watchdog():
    while True:
        time.sleep(2)
        if time.time() - state["t"] > 30:
            import numpy as np
            rec = prog.copy()
            live = np.nonzero(rec[:, 0] != -7)[0]
            print(f"WATCHDOG: step {state['step']} stuck; {len(live)} CTAs reported", flush=True)
            kinds = {}
            for i in live:
                kinds.setdefault(tuple(rec[i]), []).append(int(i))
            for k, v in sorted(kinds.items(), key=lambda kv: -len(kv[1]))[:40]:
                print("  rec", k, "ctas", v[:16], len(v), flush=True)
            os._exit(3)


if args.watch:
    threading.Thread(target=watchdog, daemon=True).start()
for k in range(93 + args.start):
    state["step"], state["t"] = -1000 + k, time.time()
    st.step_device(ptrs[t], stream.cuda_stream)
    torch.cuda.synchronize()
    t += 1
api.debug_stats(reset=True)
st.profile(True)
for k in range(args.steps):
    state["step"], state["t"] = k, time.time()
    st.step_device(ptrs[t], stream.cuda_stream)
    t += 1
    ms, steps = st.profile_read()
    st.profile(True)
    d = api.debug_stats(reset=True)
    print(f"step {k}: motion {ms[0]:.3f} ms  ccl {ms[1]:.3f} ms  meanshift {ms[2]:.3f} ms  gate+spawn {ms[3]:.3f} ms  {d}",
          flush=True)
st.profile(False)
for s in range(min(S, 4)):
    b = st.blobs(s)
    print("stream", s, "blobs", len(b), "areas", sorted(b["area"].tolist())[-5:], "tracks",
          trb.Streams.__dict__ and None)

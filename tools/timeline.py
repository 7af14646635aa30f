"""GPU timeline of a few steady steps (torch.profiler / CUPTI activity
records: every kernel and memcpy with start/end on the device clock), to
find idle gaps between the step's kernels.  Diagnostics only.
python tools/timeline.py C3 [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
from torch.profiler import ProfilerActivity, profile  # noqa: E402

import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import device_frames, recipe  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
S = 64 if name.startswith("C5") else 1
clips = [recipe("C5", s) for s in range(S)] if name.startswith("C5") else [recipe(name)]
mc = MOTION_CFG(method=1) if name == "C5MODE" else MOTION_CFG()
n = 100 + steps
stream = torch.cuda.Stream()
frames = device_frames(clips, n, stream.cuda_stream)
st = trb.Streams(S, clips[0].width, clips[0].height, 1, mc, SEG_CFG(), TRACKER_CFG())
with torch.cuda.stream(stream):
    for t in range(100):
        st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    with torch.cuda.stream(stream):
        for t in range(100, n):
            st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
        st.join(stream.cuda_stream)
    torch.cuda.synchronize()
path = f"gpurun_out/timeline_{name}.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"]
busy_end = t0
idle = 0.0
for e in ev:
    if e["ts"] > busy_end:
        idle += e["ts"] - busy_end
    busy_end = max(busy_end, e["ts"] + e["dur"])
span = busy_end - t0
print(f"{name}: {steps} steps, span {span:.0f} us ({span / steps:.1f} us/step), GPU idle {idle:.0f} us ({idle / steps:.1f} us/step)")
for e in ev[: min(len(ev), 60)]:
    print(f"{e['ts'] - t0:10.1f} {e['dur']:8.1f}  s{e.get('args', {}).get('stream', '?'):>3}  {e['name'][:60]}")

"""Host enqueue time per step vs device time (small single-stream configs are
launch/host bound when the API calls per step cost more than the kernels)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import device_frames, recipe  # noqa: E402

for name in ("C1", "C2", "C3"):
    clip = recipe(name)
    fr = device_frames([clip], 300)
    st = trb.Streams(1, clip.width, clip.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    stream = torch.cuda.Stream()
    for t in range(100):
        st.step_device([fr[0, t].data_ptr()], stream.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(stream)
    hs = []
    for t in range(100, 200):
        st.step_device([fr[0, t].data_ptr()], stream.cuda_stream)
        hs.append(time.perf_counter())
    h1 = time.perf_counter()
    first = (hs[9] - h0) / 10  # before the launch queue can fill
    st.join(stream.cuda_stream)
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"{name}: host enqueue {1e3 * (h1 - h0) / 100:.3f} ms/step (first 10 steps {1e3 * first:.3f}), "
          f"device {e0.elapsed_time(e1) / 100:.3f} ms/step")

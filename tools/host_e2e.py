"""Host cost per step of the host-frame path (trb_streams_step_host_async_out)
on the single-stream configs: Python wrapper vs the bare C call, against the
device time per step."""
import ctypes as C
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import device_frames, recipe  # noqa: E402

for name in ("C1", "C2", "C3"):
    clip = recipe(name)
    n = 300
    fr = device_frames([clip], n)
    host = torch.empty((n, clip.width * clip.height), dtype=torch.uint8).pin_memory()
    host.copy_(fr[0].reshape(n, -1))
    hn = host.numpy()
    st = trb.Streams(1, clip.width, clip.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    outs = [api.StepOutput(1, blob_cap=64, log_cap=32) for _ in range(n)]
    for t in range(100):
        st.step_host_async([hn[t]], outs[t])
    st.synchronize()
    # python wrapper
    t0 = time.perf_counter()
    for t in range(100, 200):
        st.step_host_async([hn[t]], outs[t])
    t1 = time.perf_counter()
    st.synchronize()
    t2 = time.perf_counter()
    # bare C call
    L = api.lib()
    ptrs = (C.c_void_p * 1)()
    t3 = time.perf_counter()
    for t in range(200, 300):
        ptrs[0] = hn[t].ctypes.data
        L.trb_streams_step_host_async_out(st._h, ptrs, C.byref(outs[t].c), C.c_void_p(0))
    t4 = time.perf_counter()
    st.synchronize()
    t5 = time.perf_counter()
    print(f"{name}: python enqueue {1e3 * (t1 - t0) / 100:.3f} ms/step (wall {1e3 * (t2 - t0) / 100:.3f}); "
          f"bare C enqueue {1e3 * (t4 - t3) / 100:.3f} ms/step (wall {1e3 * (t5 - t3) / 100:.3f})")

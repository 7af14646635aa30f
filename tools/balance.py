"""Load balance of the mean-shift kernel (diagnostics build): per-CTA busy
time and finish time over a few C5 steps.  Diagnostics only."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
_DIAG = os.path.join(ROOT, "paper_1310_3322_b200", "libtrb_diag.so")
if os.path.exists(_DIAG):
    os.environ.setdefault("TRB_LIB", _DIAG)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1310_3322_b200.synth import device_frames  # noqa: E402
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import recipe  # noqa: E402

S = 64
stream = torch.cuda.Stream()
clips = [recipe("C5", s) for s in range(S)]
n = 93 + 12
frames = device_frames(clips, n, stream.cuda_stream)
st = trb.Streams(S, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
for t in range(93):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
L = api.lib()
L.trb_debug_cta_times.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(2048, np.uint64)
api.debug_itlog(True)
# back-to-back steps (the bench's issue pattern, step overlap active): the
# per-CTA [busy, last end] accumulate over all steps, so also run them one by
# one below for per-step spans
L.trb_debug_cta_times(buf.ctypes.data, 1)
t_wall = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t_wall[0].record(stream)
for t in range(93, 99):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
st.join(stream.cuda_stream)
t_wall[1].record(stream)
torch.cuda.synchronize()
L.trb_debug_cta_times(buf.ctypes.data, 1)
busy = buf[0::2].astype(np.float64)
print(f"back-to-back: 6 steps in {t_wall[0].elapsed_time(t_wall[1]):.2f} ms; mean-shift CTA busy "
      f"{busy[busy > 0].mean() / 1e3 / 6:.0f} us per step per CTA")
for t in range(99, n):
    L.trb_debug_cta_times(buf.ctypes.data, 1)
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
    torch.cuda.synchronize()
    L.trb_debug_cta_times(buf.ctypes.data, 1)
    busy, end = buf[0::2].astype(np.float64), buf[1::2].astype(np.float64)
    used = end > 0
    busy, end = busy[used], end[used]
    start = (end - busy).min()
    span = (end.max() - start) / 1e3
    print(f"step {t}: {used.sum()} CTAs, kernel span ~{span:.0f} us, mean busy {busy.mean() / 1e3:.0f} us, "
          f"busy/span {busy.mean() / 1e3 / span:.2f}; finish percentiles (us) "
          + " ".join(f"{np.percentile((end - start) / 1e3, p):.0f}" for p in (10, 50, 90, 100)))
api.debug_itlog(False)

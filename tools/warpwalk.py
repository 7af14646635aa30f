"""Per (cluster rank, warp) phase-B walk time of the mean-shift engine runs
over a few steady C5 steps (diagnostics build): where the slowest warps of a
cluster sit.  Diagnostics only."""
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

S, steps = 64, 3
stream = torch.cuda.Stream()
clips = [recipe("C5", s) for s in range(S)]
n = 93 + steps
frames = device_frames(clips, n, stream.cuda_stream)
st = trb.Streams(S, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
for t in range(93):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
L = api.lib()
L.trb_debug_warp_walks.argtypes = [C.c_void_p, C.c_int]
buf = np.zeros(128, np.uint64)
L.trb_debug_warp_walks(buf.ctypes.data, 1)
api.debug_itlog(True)
for t in range(93, n):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
api.debug_itlog(False)
L.trb_debug_warp_walks(buf.ctypes.data, 1)
w = buf.astype(np.float64)
cls = ("0", "1-2", "3-5", "6-10", "11-20", "21-40", ">40")
for k, nm in enumerate(("histogram", "centroid")):
    b = w[16 * k:16 * k + 16]
    print(f"{nm}: working warps by slow-path events (sum over lanes): warps/step, mean walk us")
    for c, cn in enumerate(cls):
        n = b[2 * c + 1]
        if n:
            print(f"   {cn:>6s} {n / steps:9.0f} {b[2 * c] / n / 1.965e3:8.2f}")

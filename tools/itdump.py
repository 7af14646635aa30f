"""Dump the raw per-iteration log (item, group size, window px, cycles) of a
few steady C5 steps, one array per step, for offline schedule modelling
(diagnostics build).  python tools/itdump.py [streams] [steps] [out.npz]"""
import os
import sys

_DIAG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1310_3322_b200",
                     "libtrb_diag.so")
if os.path.exists(_DIAG):
    os.environ.setdefault("TRB_LIB", _DIAG)

import numpy as np  # noqa: E402
import torch  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1310_3322_b200.synth import device_frames  # noqa: E402
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import recipe  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 6
out = sys.argv[3] if len(sys.argv) > 3 else "gpurun_out/itdump.npz"
stream = torch.cuda.Stream()
clips = [recipe("C5", s) for s in range(S)]
n = 93 + steps
frames = device_frames(clips, n, stream.cuda_stream)
st = trb.Streams(S, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
for t in range(93):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
res = {}
for k, t in enumerate(range(93, n)):
    api.debug_itlog(True)
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
    torch.cuda.synchronize()
    a = api.debug_itlog(False)
    res[f"step{k}"] = np.stack([a[:, 0] >> 32, (a[:, 0] >> 24) & 0xff, a[:, 0] & 0xffffff, a[:, 1]], 1)
np.savez_compressed(out, **res)
print("saved", out, {k: v.shape for k, v in res.items()})

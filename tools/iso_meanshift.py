"""One mean-shift track in isolation (standalone API on an idle GPU) with the
diagnostics build: per-phase cycles of its iterations.  Diagnostics only."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
_DIAG = os.path.join(ROOT, "paper_1310_3322_b200", "libtrb_diag.so")
if os.path.exists(_DIAG):
    os.environ.setdefault("TRB_LIB", _DIAG)
import numpy as np  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402

W, H = 1920, 1080
size = int(sys.argv[1]) if len(sys.argv) > 1 else 40
frame = np.full((H, W), 16, np.uint8)
frame[500:500 + size, 900:900 + size] = 200
frame[500 + size // 3:500 + size, 900 + size // 4:900 + size] = 150
centers = np.array([[16.0] * 3, [150.0] * 3, [200.0] * 3] + [[float(v)] * 3 for v in range(30, 250, 17)])[:16]
target = api.histogram(frame, W, H, 1, 900 + size / 2 - 3.3, 500 + size / 2 - 2.1, size, size, centers)
api.debug_itlog(True)
for rep in range(20):
    api.meanshift_step(frame, W, H, 1, 900 + size / 2 + 4.7, 500 + size / 2 + 3.9, size, size, centers, target)
ph = api.debug_phases()
a = api.debug_itlog(False)
names = {1: "fill_u2", 2: "bin+count", 3: "count scan+sync", 4: "bin offsets", 5: "scatter+sync", 6: "bc/wsq",
         30: "div/hypot"}
for b, nm in ((7, "hist"), (18, "cent")):
    for st, what in enumerate(["A local", "A sync", "A gather+xP", "B walk", "C scan", "C sync", "C fold", "rank",
                               "rank sync", "D replay", "end sync"], start=1):
        names[b + st] = f"{nm} {what}"
it = ph[:, 0].sum()
print(f"window {size}x{size}: {it} iterations, {len(a)} logged")
tot = 0
for k in range(1, 40):
    v = ph[:, k].sum()
    if v:
        tot += v
        print(f"  {k:2d} {names.get(k, '?'):22s} {v / it / 1.9e3:8.2f} us")
print(f"  total {tot / it / 1.9e3:.2f} us per iteration")
w = ph[:, 40:56].sum(axis=0)
print(f"  walk per thread: hist {w[1] / max(1, w[12]) / 1.9e3:.2f} us, cent {w[3] / max(1, w[13]) / 1.9e3:.2f} us; "
      f"startup hist {w[14] / max(1, w[12]) / 1.9e3:.2f} cent {w[15] / max(1, w[13]) / 1.9e3:.2f}")
tr = api.debug_phases()[3, :32]  # g_phase[192..223]: last centroid walk of thread 0
print("thread 100 of CTA 1, centroid walk, cycles at each element (last run):", [int(x) for x in tr[:20]])

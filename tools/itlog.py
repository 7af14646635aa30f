"""Per mean-shift-iteration latency vs window size (diagnostics)."""
import os
import sys

# the diagnostics build of the library (make -C paper_1310_3322_b200/csrc diag)
_DIAG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1310_3322_b200",
                     "libtrb_diag.so")
if os.path.exists(_DIAG):
    os.environ.setdefault("TRB_LIB", _DIAG)

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_1310_3322_b200.synth import device_frames  # noqa: E402
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200 import api  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import recipe  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 64
steps = 4
stream = torch.cuda.Stream()
clips = [recipe("C5", s) for s in range(S)]
n = 93 + steps
frames = device_frames(clips, n, stream.cuda_stream)
st = trb.Streams(S, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
for t in range(93):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
api.debug_itlog(True)
for t in range(93, n):
    st.step_device([frames[s, t].data_ptr() for s in range(S)], stream.cuda_stream)
torch.cuda.synchronize()
ph = api.debug_phases()
a = api.debug_itlog(False)
item = (a[:, 0] >> 32)
N, cyc = (a[:, 0] & 0xffffff).astype(float), a[:, 1].astype(float)
grp = (a[:, 0] >> 24) & 0xff
# per-track totals (a track = item within a step; steps are not separated, so
# report per (item) sums divided by steps as a proxy)
tot = {}
for it, c, n_ in zip(item, cyc, N):
    t = tot.setdefault(int(it), [0.0, 0, 0.0])
    t[0] += c
    t[1] += 1
    t[2] = max(t[2], n_)
top = sorted(tot.items(), key=lambda kv: -kv[1][0])[:8]
for it, (c, k, n_) in top:
    print(f"track item {it}: {k/steps:5.1f} iters/step, {c/1.9e3/steps:8.1f} us/step, max N {n_:.0f}")
print("iterations", len(a), "per step", len(a) / steps)
for gs in sorted(set(grp.tolist())):
    m = grp == gs
    A = np.vstack([np.ones_like(N[m]), N[m]]).T
    coef, *_ = np.linalg.lstsq(A, cyc[m], rcond=None)
    print(f"group of {gs} CTAs: {m.sum()} iters, cycles ~= {coef[0]:.0f} + {coef[1]:.3f} * N"
          f"   (us: {coef[0]/1.9e3:.1f} + {coef[1]/1.9e3*1e3:.3f}/kpx)")
for lo, hi in [(0, 5e3), (5e3, 2e4), (2e4, 6e4), (6e4, 1.5e5), (1.5e5, 1e7)]:
    m = (N >= lo) & (N < hi)
    if m.any():
        print(f"N in [{lo:.0f},{hi:.0f}): {m.sum():5d} iters, mean N {N[m].mean():9.0f}, mean {cyc[m].mean()/1.9e3:8.1f} us")
print("total iteration-time (cluster-us) per step:", cyc.sum() / 1.9e3 / steps, " max N", N.max())

names = {1: "fill_u2", 2: "bin+count", 3: "count scan+sync", 4: "bin offsets", 5: "scatter+sync",
         6: "bhattacharyya/wsq", 30: "centroid div/hypot"}
for b, nm in ((7, "hist"), (18, "cent")):
    for st, what in enumerate(["A local", "A sync", "A gather+xP", "B walk", "C scan", "C sync", "C fold",
                               "rank", "rank sync", "D replay", "end sync"], start=1):
        names[b + st] = f"{nm} {what}"
names.update({31: "hist C warp scan", 32: "hist C barrier", 33: "cent C warp scan", 34: "cent C barrier"})
walk = ph[:, 40:56].copy()
ph[:, 40:56] = 0
bnames = ("<5k px", "5k-50k px", "50k-150k px", ">150k px")
print("phase us per iteration by window-size bucket:")
print(f"  {'phase':24s}" + "".join(f"{b:>13s}" for b in bnames))
cnt = np.maximum(ph[:, 0].astype(float), 1)
print(f"  {'iterations/step':24s}" + "".join(f"{c / steps:13.1f}" for c in ph[:, 0]))
for k in range(1, 64):
    if ph[:, k].any():
        print(f"  {k:2d} {names.get(k, '?'):21s}" + "".join(f"{ph[b, k] / cnt[b] / 1.9e3:13.2f}" for b in range(4)))
print(f"  {'total':24s}" + "".join(f"{ph[b, 1:].sum() / cnt[b] / 1.9e3:13.2f}" for b in range(4)))
print("per-thread B walk (rank-0 CTA threads with work): max cycles over the run, sum")
for b in range(4):
    print(f"  {bnames[b]:12s} hist max {walk[b,0]/1.9e3:9.1f} us  cent max {walk[b,2]/1.9e3:9.1f} us  "
          f"hist sum/iter {walk[b,1]/cnt[b]/1.9e3:9.1f}  cent sum/iter {walk[b,3]/cnt[b]/1.9e3:9.1f} us")
print("slow-path events per walking thread (rank-0 CTAs): max / mean arming+bp checks, max / mean breakpoints")
for b in range(4):
    w = walk[b]
    nt1, nt3 = max(1, w[12]), max(1, w[13])
    print(f"  {bnames[b]:12s} hist slow {w[4]:5d} / {w[5]/nt1:6.2f}  bp {w[6]:5d} / {w[7]/nt1:6.2f}   "
          f"cent slow {w[8]:5d} / {w[9]/nt3:6.2f}  bp {w[10]:5d} / {w[11]/nt3:6.2f}")
print("cursor start-up (walk begin -> first element's data), mean per walking thread")
for b in range(4):
    w = walk[b]
    nt1, nt3 = max(1, w[12]), max(1, w[13])
    print(f"  {bnames[b]:12s} hist {w[14]/nt1/1.9e3:7.2f} us   cent {w[15]/nt3/1.9e3:7.2f} us")

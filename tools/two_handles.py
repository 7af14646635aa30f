"""A/B: the C5 workload (64 x 1080p streams) as one handle of 64 streams vs
H handles of 64/H streams stepped alternately on their own CUDA streams
(their tracker tails overlap each other's bulk).  python tools/two_handles.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_1310_3322_b200.synth import device_frames  # noqa: E402
import paper_1310_3322_b200 as trb  # noqa: E402
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG  # noqa: E402
from paper_1310_3322_b200.synth import recipe  # noqa: E402

S, K = 64, 10
clips = [recipe("C5", s) for s in range(S)]
base = torch.cuda.Stream()
frames = bench.make_frames(trb, clips, 93 + 3 + K, base)
for H in (1, 2, 1, 2, 1, 2, 4):
    per = S // H
    hs = [trb.Streams(per, 1920, 1080, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG()) for _ in range(H)]
    cs = [torch.cuda.Stream() for _ in range(H)]
    def step(t):
        for h in range(H):
            hs[h].step_device([frames[h * per + s, t].data_ptr() for s in range(per)], cs[h].cuda_stream)
    for t in range(93 + 3):
        step(t)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(base)
    for h in range(H):
        cs[h].wait_event(e0)
    for t in range(93 + 3, 93 + 3 + K):
        step(t)
    for h in range(H):
        hs[h].join(cs[h].cuda_stream)
        base.wait_stream(cs[h])
    e1.record(base)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"H={H}: {S * K / (ms / 1e3):.0f} frames/s ({ms / K:.2f} ms/step)", flush=True)
    del hs
    torch.cuda.synchronize()

#!/bin/bash
# C5 with fewer streams per GPU: which cluster size wins (TRB_CLUSTER fixed), plus the active-track count
cd "$(dirname "$0")/.."
for S in ${SS:-4 8 16 32}; do for g in 8 12 16; do
  TRB_CLUSTER=$g timeout 300 python bench.py --streams $S --steps 20 --warmup 5 --no-cpu-baseline --no-e2e \
    --verify-streams 0 > gpurun_out/ab.json 2> gpurun_out/ab.err
  echo "S=$S G=$g :: $(python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print(round(d['value']), round(d['ms_per_step'],3))" 2>&1 | tail -1)"
done; done
python - <<'PY'
import os, sys
sys.path.insert(0, '.')
import paper_1310_3322_b200 as trb
from paper_1310_3322_b200.abi import MOTION_CFG, SEG_CFG, TRACKER_CFG
from paper_1310_3322_b200.synth import device_frames, recipe
for cfg, S in (("C4", 1), ("C5", 4)):
    clips = [recipe(cfg, s) for s in range(S)] if cfg == "C5" else [recipe("C4")]
    fr = device_frames(clips, 115)
    c0 = clips[0]
    st = trb.Streams(S, c0.width, c0.height, 1, MOTION_CFG(), SEG_CFG(), TRACKER_CFG())
    for t in range(115):
        st.step_device([fr[s, t].data_ptr() for s in range(S)])
    st.synchronize()
    n = sum(st.num_tracks(s) for s in range(S))
    print(cfg, "streams", S, "tracks listed at frame 114:", n, [len(st.log(s)) for s in range(S)])
PY

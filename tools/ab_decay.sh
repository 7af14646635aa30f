#!/bin/bash
# A/B: decaying-maximum iteration hint for the mean-shift queue order
cd "$(dirname "$0")/.."
for cfg in C5 C4; do for rep in 1 2 3; do for kv in "TRB_ITER_DECAY=0" "TRB_ITER_DECAY=1" "TRB_ITER_DECAY=2" "TRB_ITER_DECAY=4"; do
  env $kv timeout 300 python bench.py --config $cfg --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$cfg $kv', round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3))"
done; done; done

#!/bin/bash
# A/B: mean-shift cluster count on C5MODE (the Mode motion kernel needs SMs beside the tracker)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for kv in "TRB_TRACK_CLUSTERS=33" "TRB_TRACK_CLUSTERS=29" "TRB_TRACK_CLUSTERS=25" "TRB_TRACK_CLUSTERS=21" "TRB_OVERLAP=0"; do
  env $kv timeout 300 python bench.py --config C5MODE --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3))"
done; done

#!/bin/bash
# A/B: mean-shift cluster count (SMs left to the overlapped motion + CCL of the next step)
cd "$(dirname "$0")/.."
for rep in 1 2; do
for kv in "TRB_TRACK_CLUSTERS=33" "TRB_TRACK_CLUSTERS=31" "TRB_TRACK_CLUSTERS=29" "TRB_TRACK_CLUSTERS=27" "TRB_TRACK_CLUSTERS=24" "TRB_OVERLAP=0"; do
  env $kv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-e2e --verify-streams 0 \
    > gpurun_out/ab.json 2>/dev/null
  python -c "import json;d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]);print('$kv', round(d['value']), round(d['ms_per_step'],3), round(d['config']['stage_ms_per_step']['track_meanshift'],3))"
done; done
